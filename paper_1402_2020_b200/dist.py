"""Multi-GPU partitions of the matching path (one process per GPU).

Two partitions, both implemented in the C ABI over
NCCL (include/bsm_cuda.h "Multi-GPU", csrc/bsm_dist.cuh); this module is the
thin Python caller:

* batch of pairs (BASELINE configs[3]): pairs are independent units, sharded
  contiguously over ranks (``shard_units``); no data-path collective; the
  refined maps are gathered to one root rank at the end
  (``bsm_pipeline_pairs_sharded_u8``: ncclSend / ncclRecv).
* one large frame (configs[4]): contiguous row bands (``band_rows``).  Every
  rank holds both full views and computes its band with a vote-radius halo of
  redundant rows, so the only exchange is the final all-gather of the refined
  bands (``bsm_pipeline_frame_bands_u8``: ncclAllGather), or, with
  ``transport="p2p"``, no collective at all: the check and refine kernels
  store the band into every rank's map over peer memory (``bsm_frame``).  A band-local
  ``max_bin`` is safe: bins above it are 0 for every pixel of the band and
  cannot win the strict-'>' argmax (refine.hpp:102-105).

``torch.distributed`` is the plumbing: it carries the NCCL unique id from rank
0 to the others.  With a non-NCCL process group (gloo: several processes
sharing one GPU in the tests, or hosts without NCCL) the same per-rank compute
runs through the C ABI (``run_pipeline_band`` / ``run_pipeline_batch``) and
the bands / maps travel through the group's own all-gather instead.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import (BsmConfig, Context, DisparityMap, SamplingPattern, _params, _ptr_array, _u8, default_context,
               generate_pattern, run_pipeline_band, run_pipeline_batch)
from ._lib import DimensionMismatch, check, lib


def band_rows(height: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous row band [y0, y1) of `rank`; band sizes differ by at most 1
    (the same formula as csrc/bsm_dist.cuh band_of)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    base, extra = divmod(height, world)
    y0 = rank * base + min(rank, extra)
    return y0, y0 + base + (1 if rank < extra else 0)


def shard_units(n_units: int, world: int, rank: int) -> range:
    """Contiguous shard of unit indices owned by `rank`."""
    y0, y1 = band_rows(n_units, world, rank)
    return range(y0, y1)


class Comm:
    """A bsm_comm (NCCL communicator bound to a context) for this rank of a
    torch.distributed group; the NCCL unique id travels through the group."""

    def __init__(self, ctx: Optional[Context] = None, group=None):
        import torch.distributed as dist
        self.ctx = ctx or default_context()
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        uid = (C.c_uint8 * 128)()
        if self.rank == 0:
            check(lib().bsm_comm_unique_id(uid))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
        h = C.c_void_p()
        check(lib().bsm_comm_create(self.ctx.handle, uid, self.world, self.rank, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().bsm_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _is_nccl(group) -> bool:
    import torch.distributed as dist
    return dist.get_backend(group) == "nccl"


def _comm_for(ctx: Context, group) -> Comm:
    cache = ctx.__dict__.setdefault("_comms", {})
    key = id(group)
    if key not in cache:
        cache[key] = Comm(ctx, group)
    return cache[key]


def allgather_bands(band: DisparityMap, height: int, group=None) -> DisparityMap:
    """All-gather row bands (equal-or-off-by-one heights) into the full map
    through the group's own collective (the non-NCCL path)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if _is_nccl(group) else torch.device("cpu")
    W = band.width
    rows_max = -(-height // world)
    d = torch.zeros((rows_max, W), dtype=torch.float32, device=dev)
    v = torch.zeros((rows_max, W), dtype=torch.uint8, device=dev)
    d[: band.height] = torch.from_numpy(np.ascontiguousarray(band.disparity)).to(dev)
    v[: band.height] = torch.from_numpy(np.ascontiguousarray(band.valid)).to(dev)
    ds = [torch.empty_like(d) for _ in range(world)]
    vs = [torch.empty_like(v) for _ in range(world)]
    dist.all_gather(ds, d, group=group)
    dist.all_gather(vs, v, group=group)
    out_d = np.empty((height, W), np.float32)
    out_v = np.empty((height, W), np.uint8)
    for r in range(world):
        y0, y1 = band_rows(height, world, r)
        out_d[y0:y1] = ds[r][: y1 - y0].cpu().numpy()
        out_v[y0:y1] = vs[r][: y1 - y0].cpu().numpy()
    return DisparityMap(out_d, out_v)


def gather_pairs(results: List[Tuple[int, DisparityMap]], n_units: int, shape: Tuple[int, int], dst: int = 0,
                 group=None) -> Optional[List[DisparityMap]]:
    """Gather every rank's (index, map) results to rank `dst` (None elsewhere)
    through the group's own collective (the non-NCCL path)."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if _is_nccl(group) else torch.device("cpu")
    H, W = shape
    per = max(len(shard_units(n_units, world, r)) for r in range(world))
    d = torch.zeros((per, H, W), dtype=torch.float32, device=dev)
    v = torch.zeros((per, H, W), dtype=torch.uint8, device=dev)
    for k, (_, m) in enumerate(results):
        d[k] = torch.from_numpy(m.disparity).to(dev)
        v[k] = torch.from_numpy(m.valid).to(dev)
    ds = [torch.empty_like(d) for _ in range(world)]
    vs = [torch.empty_like(v) for _ in range(world)]
    dist.all_gather(ds, d, group=group)
    dist.all_gather(vs, v, group=group)
    if rank != dst:
        return None
    out: List[Optional[DisparityMap]] = [None] * n_units
    for r in range(world):
        for k, i in enumerate(shard_units(n_units, world, r)):
            out[i] = DisparityMap(ds[r][k].cpu().numpy(), vs[r][k].cpu().numpy())
    return out  # type: ignore[return-value]


class Frame:
    """A bsm_frame: this rank's full-frame refined map in device memory,
    exported through CUDA IPC and attached to every other rank's map (the
    handles travel through the torch.distributed group)."""

    def __init__(self, ctx: Context, W: int, H: int, group=None):
        import torch.distributed as dist
        self.ctx = ctx
        self.W, self.H = W, H
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        h = C.c_void_p()
        handle = (C.c_uint8 * 128)()
        check(lib().bsm_frame_create(ctx.handle, W, H, self.world, self.rank, C.byref(h), handle))
        self._h = h
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(handle), group=group)
        allh = (C.c_uint8 * (128 * self.world)).from_buffer_copy(b"".join(handles))
        check(lib().bsm_frame_attach(self._h, allh))

    def fetch(self) -> DisparityMap:
        d = np.empty((self.H, self.W), np.float32)
        v = np.empty((self.H, self.W), np.uint8)
        check(lib().bsm_frame_fetch(self._h, d.ctypes.data, v.ctypes.data))
        return DisparityMap(d, v)

    def close(self):
        if getattr(self, "_h", None):
            lib().bsm_frame_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_frame_bands(left, right, cfg: BsmConfig, pattern: Optional[SamplingPattern] = None, group=None,
                    ctx: Optional[Context] = None, transport: str = "auto") -> DisparityMap:
    """run_pipeline(...).refined of one frame, row-band partitioned over the
    group; every rank returns the whole refined map.

    transport: "nccl" (bsm_pipeline_frame_bands_u8: one ncclAllGather of the
    bands), "p2p" (bsm_frame: the check and refine kernels store each band
    straight into every rank's map over peer memory; one barrier), "group"
    (the band through run_pipeline_band, gathered by the group's own
    collective); "auto" = "nccl" with an NCCL group, else "group"."""
    import torch.distributed as dist
    L, R = _u8(left, "left"), _u8(right, "right")
    if L.shape != R.shape:
        raise DimensionMismatch("pipeline: left/right dimensions differ")
    cfg.validate()
    pattern = pattern or generate_pattern(cfg=cfg)
    ctx = ctx or default_context()
    H, W = L.shape
    if transport == "auto":
        transport = "nccl" if _is_nccl(group) else "group"
    if transport == "p2p":
        ctx.set_pattern(pattern)
        frame = Frame(ctx, W, H, group)
        try:
            p = _params(cfg)
            check(lib().bsm_pipeline_frame_bands_p2p_u8(ctx.handle, frame._h, L.ctypes.data, R.ctypes.data,
                                                        C.byref(p)))
            dist.barrier(group=group)  # every rank's stores have completed
            return frame.fetch()
        finally:
            dist.barrier(group=group)  # no rank unmaps a frame another rank still writes
            frame.close()
    if transport == "nccl":
        ctx.set_pattern(pattern)
        comm = _comm_for(ctx, group)
        d = np.empty((H, W), np.float32)
        v = np.empty((H, W), np.uint8)
        p = _params(cfg)
        check(lib().bsm_pipeline_frame_bands_u8(ctx.handle, comm.handle, L.ctypes.data, R.ctypes.data, W, H,
                                                C.byref(p), d.ctypes.data, v.ctypes.data))
        return DisparityMap(d, v)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    y0, y1 = band_rows(H, world, rank)
    band = run_pipeline_band(L, R, cfg, y0, y1, pattern=pattern, ctx=ctx)
    return allgather_bands(band, H, group)


def run_pairs_sharded(pairs: Sequence[Tuple[np.ndarray, np.ndarray]], cfg: BsmConfig,
                      pattern: Optional[SamplingPattern] = None, group=None, ctx: Optional[Context] = None,
                      root: int = 0) -> Optional[List[DisparityMap]]:
    """run_pipeline(...).refined of every pair of a batch, pairs sharded over
    the group; the list of all maps on rank `root`, None on the others.  Only
    this rank's shard of `pairs` is read."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n = len(pairs)
    mine = shard_units(n, world, rank)
    cfg.validate()
    pattern = pattern or generate_pattern(cfg=cfg)
    ctx = ctx or default_context()
    views = {i: (_u8(pairs[i][0], "left"), _u8(pairs[i][1], "right")) for i in mine}
    shapes = {v[0].shape for v in views.values()} | {v[1].shape for v in views.values()}
    if len(shapes) > 1:
        raise DimensionMismatch("pipeline: left/right dimensions differ")
    H, W = np.asarray(pairs[0][0]).shape
    if _is_nccl(group):
        ctx.set_pattern(pattern)
        comm = _comm_for(ctx, group)
        blank = np.zeros((1, 1), np.uint8)
        lefts = [views[i][0] if i in views else blank for i in range(n)]
        rights = [views[i][1] if i in views else blank for i in range(n)]
        outs = ([(np.empty((H, W), np.float32), np.empty((H, W), np.uint8)) for _ in range(n)]
                if rank == root else None)
        p = _params(cfg)
        check(lib().bsm_pipeline_pairs_sharded_u8(
            ctx.handle, comm.handle, n, _ptr_array(lefts), _ptr_array(rights), W, H, C.byref(p), root,
            _ptr_array([o[0] for o in outs]) if outs else None, _ptr_array([o[1] for o in outs]) if outs else None))
        return [DisparityMap(d, v) for d, v in outs] if outs else None
    maps = run_pipeline_batch([views[i] for i in mine], cfg, pattern=pattern, ctx=ctx)
    return gather_pairs(list(zip(mine, maps)), n, (H, W), dst=root, group=group)
