"""Multi-process (gloo, world_size 2, CPU) tests of the multi-GPU partition
and gather logic (paper_1402_2020_b200.dist).  The per-unit compute is the
C restatement (test infrastructure); the GPU halo computation itself is
covered by tests/test_gpu_parity.py::test_band_matches_full."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1402_2020_b200.dist import band_rows, shard_units


def test_band_rows_partition():
    for H in (1, 7, 375, 2160):
        for world in (1, 2, 3, 4, 8):
            if world > H:
                continue
            rows = [band_rows(H, world, r) for r in range(world)]
            assert rows[0][0] == 0 and rows[-1][1] == H
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
            sizes = [b - a for a, b in rows]
            assert max(sizes) - min(sizes) <= 1
    assert band_rows(2160, 8, 3) == (810, 1080)
    assert list(shard_units(64, 8, 7)) == list(range(56, 64))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, q):
    import sys
    ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_1402_2020_b200 as bsm
        from paper_1402_2020_b200 import dist as bd
        from paper_1402_2020_b200.synth import workload_pair
        orc = oracle.Restatement()
        pairs_arr = orc.generate_pattern(256, 10, 2.5, 7)
        pattern = bsm.SamplingPattern(256, 10, 2.5, 7, pairs_arr)
        cfg = bsm.BsmConfig(n=256, window=10, spread=2.5, seed=7, d_max=24, vote_radius=4)

        def full(L, R):
            o = orc.pipeline_u8(L, R, pairs_arr, 10, 24, radius=4)
            return bsm.DisparityMap(o["refined_d"], o["refined_v"])

        if kind == "bands":
            left, right = workload_pair("c1")
            L, R = left[100:133, 100:180].copy(), right[100:133, 100:180].copy()
            ref_full = full(L, R)
            got = bd.run_frame_bands(L, R, cfg, pattern,
                                     compute_band=lambda L_, R_, c, y0, y1, p: bsm.DisparityMap(
                                         ref_full.disparity[y0:y1], ref_full.valid[y0:y1]))
            q.put((rank, got == ref_full))
        else:
            pairs = []
            for i in range(5):
                left, right = workload_pair("c1", index=i)
                pairs.append((left[50:70, 30:90].copy(), right[50:70, 30:90].copy()))
            mine = bd.run_pairs_sharded(pairs, cfg, pattern, compute_pair=lambda L, R, c, p: full(L, R))
            assert [i for i, _ in mine] == list(bd.shard_units(5, world, rank))
            out = bd.gather_pairs(mine, 5, (20, 60), dst=0)
            if rank == 0:
                ok = all(out[i] == full(*pairs[i]) for i in range(5))
                q.put((rank, ok))
            else:
                q.put((rank, out is None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["bands", "pairs"])
def test_gloo_world2(kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
