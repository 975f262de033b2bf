"""Multi-GPU partitions of the matching path (one process per GPU).

Two partitions:

* batch of pairs (BASELINE configs[3]): pairs are independent units, sharded
  contiguously over ranks; no data-path collective; results are gathered to
  one rank only at the end (``gather_pairs``).
* one large frame (configs[4]): contiguous row bands.  Every rank holds both
  full views and computes its band with a vote-radius halo of redundant rows
  (``run_pipeline_band``), so the only exchange is the final all-gather of
  the refined bands.  A band-local ``max_bin`` is safe: bins above it are 0
  for every pixel of the band and cannot win the strict-'>' argmax
  (refine.hpp:102-105).

Rendezvous/plumbing is ``torch.distributed`` (NCCL over NVLink on GPUs, gloo
for the CPU tests).  The compute of a unit is injectable so the partition and
gather logic can be tested on CPU against the checker.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import BsmConfig, DisparityMap, SamplingPattern, run_pipeline, run_pipeline_band


def band_rows(height: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous row band [y0, y1) of `rank`; band sizes differ by at most 1."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    base, extra = divmod(height, world)
    y0 = rank * base + min(rank, extra)
    return y0, y0 + base + (1 if rank < extra else 0)


def shard_units(n_units: int, world: int, rank: int) -> range:
    """Contiguous shard of unit indices owned by `rank`."""
    y0, y1 = band_rows(n_units, world, rank)
    return range(y0, y1)


def _device_for(backend: str):
    import torch
    if backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def allgather_bands(band: DisparityMap, height: int, group=None) -> DisparityMap:
    """All-gather row bands (equal-or-off-by-one heights) into the full map."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = _device_for(dist.get_backend(group))
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


def run_frame_bands(left, right, cfg: BsmConfig, pattern: Optional[SamplingPattern] = None, group=None,
                    compute_band: Optional[Callable] = None) -> DisparityMap:
    """run_pipeline(...).refined of one frame, row-band partitioned over the group."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    H = np.asarray(left).shape[0]
    y0, y1 = band_rows(H, world, rank)
    fn = compute_band or (lambda L, R, c, a, b, p: run_pipeline_band(L, R, c, a, b, pattern=p))
    band = fn(left, right, cfg, y0, y1, pattern)
    return allgather_bands(band, H, group)


def run_pairs_sharded(pairs: Sequence[Tuple[np.ndarray, np.ndarray]], cfg: BsmConfig,
                      pattern: Optional[SamplingPattern] = None, group=None,
                      compute_pair: Optional[Callable] = None) -> List[Tuple[int, DisparityMap]]:
    """Refined maps of this rank's shard of a batch of pairs (no collective)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    fn = compute_pair or (lambda L, R, c, p: run_pipeline(L, R, c, p, outputs="refined").refined)
    return [(i, fn(pairs[i][0], pairs[i][1], cfg, pattern)) for i in shard_units(len(pairs), world, rank)]


def gather_pairs(results: List[Tuple[int, DisparityMap]], n_units: int, shape: Tuple[int, int], dst: int = 0,
                 group=None) -> Optional[List[DisparityMap]]:
    """Gather every rank's (index, map) results to rank `dst` (None elsewhere)."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = _device_for(dist.get_backend(group))
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
