"""Multi-process tests of the multi-GPU partitions (paper_1402_2020_b200.dist,
csrc/bsm_dist.cuh).

* CPU (gloo, world 2): the partition arithmetic and the gather helpers of the
  non-NCCL path, on synthetic maps -- these test the gathers only.
* GPU (gloo, world 2, both processes on cuda:0 with their own context): the
  REAL band / batch compute through the C ABI in two processes, assembled and
  compared with the reference's maps (committed goldens of c5 and c4) -- the
  worker-count independence the reference guarantees (parallel.hpp:12-14,
  test_pipeline.cpp:42-63).  Only one GPU exists here, and NCCL refuses two
  ranks on one device, so the NCCL entry points are run at world 1
  (test_nccl_world1): the same code path with a one-rank communicator.
"""
import hashlib
import json
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1402_2020_b200.dist import band_rows, shard_units

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


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
    assert [len(shard_units(5, 2, r)) for r in range(2)] == [3, 2]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(target, world, *args, timeout=600):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=timeout) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    return res


def _init(rank, world, port, backend):
    import sys
    ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group(backend, rank=rank, world_size=world)
    return dist


# --------------------------------------------------------------------------
# CPU: gather helpers of the non-NCCL path (synthetic maps, no compute)
def _gather_worker(rank, world, port, q, kind):
    dist = _init(rank, world, port, "gloo")
    try:
        import paper_1402_2020_b200 as bsm
        from paper_1402_2020_b200 import dist as bd
        rng = np.random.default_rng(5)
        if kind == "bands":
            full = bsm.DisparityMap(rng.random((13, 17), dtype=np.float32), rng.integers(0, 2, (13, 17), np.uint8))
            y0, y1 = band_rows(13, world, rank)
            got = bd.allgather_bands(bsm.DisparityMap(full.disparity[y0:y1], full.valid[y0:y1]), 13)
            q.put((rank, got == full))
        else:
            maps = [bsm.DisparityMap(rng.random((4, 6), dtype=np.float32), rng.integers(0, 2, (4, 6), np.uint8))
                    for _ in range(5)]
            mine = [(i, maps[i]) for i in shard_units(5, world, rank)]
            out = bd.gather_pairs(mine, 5, (4, 6), dst=0)
            q.put((rank, all(a == b for a, b in zip(out, maps)) if rank == 0 else out is None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["bands", "pairs"])
def test_gather_helpers_gloo_world2(kind):
    assert _spawn(_gather_worker, 2, kind, timeout=240) == {0: True, 1: True}


# --------------------------------------------------------------------------
# GPU: real compute in two processes (gloo gathers), against the reference
def _compute_worker(rank, world, port, q, kind):
    dist = _init(rank, world, port, "gloo")
    try:
        import paper_1402_2020_b200 as bsm
        from paper_1402_2020_b200 import dist as bd
        from paper_1402_2020_b200.synth import workload_pair
        ctx = bsm.Context(0)
        if kind in ("bands", "p2p"):
            g = json.load(open(os.path.join(GOLDEN, "c5.json")))
            left, right = workload_pair("c5")
            m = bd.run_frame_bands(left, right, bsm.BsmConfig(d_max=g["d_max"]), ctx=ctx,
                                   transport="p2p" if kind == "p2p" else "auto")
            q.put((rank, sha(m.disparity) == g["maps"]["refined_d"] and sha(m.valid) == g["maps"]["refined_v"]))
        else:
            gs = [json.load(open(os.path.join(GOLDEN, f"c4_{i}.json"))) for i in range(5)]
            pairs = [workload_pair("c4", index=i) if i in shard_units(5, world, rank) else (None, None)
                     for i in range(5)]
            pairs = [(l, r) if l is not None else pairs[min(shard_units(5, world, rank))] for l, r in pairs]
            out = bd.run_pairs_sharded(pairs, bsm.BsmConfig(d_max=192), ctx=ctx, root=0)
            if rank == 0:
                q.put((rank, all(sha(m.disparity) == g["maps"]["refined_d"] and sha(m.valid) == g["maps"]["refined_v"]
                                 for m, g in zip(out, gs))))
            else:
                q.put((rank, out is None))
    except Exception as e:  # report instead of hanging the queue
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["bands", "pairs", "p2p"])
def test_real_compute_world2_matches_reference(kind):
    """p2p: the two processes map each other's full-frame maps (CUDA IPC) and
    their check / refine kernels store each band into both (bsm_frame); no
    kernel waits on the other process -- the barrier is on the host."""
    need = ["c5"] if kind in ("bands", "p2p") else [f"c4_{i}" for i in range(5)]
    if not all(os.path.exists(os.path.join(GOLDEN, f"{t}.json")) for t in need):
        pytest.skip("goldens not generated")
    assert _spawn(_compute_worker, 2, kind) == {0: True, 1: True}


def _nccl_worker(rank, world, port, q):
    dist = _init(rank, world, port, "nccl")
    try:
        import torch
        torch.cuda.set_device(0)
        import paper_1402_2020_b200 as bsm
        from paper_1402_2020_b200 import dist as bd
        from paper_1402_2020_b200.synth import workload_pair
        ctx = bsm.Context(0)
        g = json.load(open(os.path.join(GOLDEN, "c5.json")))
        left, right = workload_pair("c5")
        m = bd.run_frame_bands(left, right, bsm.BsmConfig(d_max=g["d_max"]), ctx=ctx)
        ok_bands = sha(m.disparity) == g["maps"]["refined_d"] and sha(m.valid) == g["maps"]["refined_v"]
        gs = [json.load(open(os.path.join(GOLDEN, f"c4_{i}.json"))) for i in range(3)]
        out = bd.run_pairs_sharded([workload_pair("c4", index=i) for i in range(3)], bsm.BsmConfig(d_max=192),
                                   ctx=ctx, root=0)
        ok_pairs = all(sha(o.disparity) == gg["maps"]["refined_d"] and sha(o.valid) == gg["maps"]["refined_v"]
                       for o, gg in zip(out, gs))
        ctx.close()
        q.put((rank, (ok_bands, ok_pairs)))
    except Exception as e:
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_world1():
    """The C-ABI NCCL entry points (bsm_comm_*, frame bands all-gather,
    sharded pairs send/recv) with a one-rank NCCL group."""
    if not all(os.path.exists(os.path.join(GOLDEN, f"{t}.json")) for t in ["c5", "c4_0", "c4_1", "c4_2"]):
        pytest.skip("goldens not generated")
    assert _spawn(_nccl_worker, 1) == {0: (True, True)}
