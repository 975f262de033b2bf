#!/usr/bin/env python
"""Benchmark of the Binary Stereo Matching hot path on B200.

metric: Mdisp-evals/s = W*H*D per second (BASELINE.json), whole job.

Default workload: BASELINE.json configs[3] -- a batch of 64 synthetic
1920x1080 pairs, D=192, the config the metric's "1/2/4/8 B200" is quoted on.
One step = run_pipeline (descriptors + masks of both views, masked WTA in both
directions, left/right check, voting refinement) of ALL 64 pairs; with N
ranks (torchrun) rank r matches pairs shard_units(64, N, r) -- independent
units, fixed total work (strong scaling), no data-path collective.
`--workload c5` at N > 1 is the row-band partition of configs[4] (one NCCL
all-gather of the refined bands); the single-pair configs (c1, c2, c3, c2rgb)
run one pair per rank (replicas).

  value   device-resident views (inputs in HBM before the timed region),
          CUDA events on the library's stream; a 256 MiB L2 flush before each
          step (outside the events)
  e2e     the public C-ABI call a user makes (bsm_pipeline_batch_u8 for the
          batch, bsm_pipeline_u8 / _rgb for one pair) with pinned HOST
          buffers: the H2D of every view and the D2H of every refined map
          (float + valid) are inside the timed region
  roofline  the dominant kernel of the step (largest measured stage time):
          `roofline_cost` is the fused cost + WTA kernel (K3, tensor cores)
          against the live dense FP4 MMA rate of this GPU (algorithmic flops:
          one MAC per descriptor bit per in-bounds evaluation), beside it the
          MMA's busy fraction (band waste included), the shared-memory
          bandwidth that binds it, and the same work as popcount word-ops
          against the integer-pipe roofline; `roofline_mask` is the mask
          kernel (K2) against its shared-memory gather floor
  cpu_baseline  the reference library compiled in place (oracle/_ref), all
          host threads, median of repeated runs on a row band of pair 0
  cold_start  context creation + pattern upload + first pipeline (tables)

--impl reference: the reference CPU implementation alone (rank 0), same
metric and config; the K timed steps walk down pair 0 of the workload in
consecutive row bands (each band run through run_pipeline as its own image,
at least 8 rows per host thread), covering the whole frame when K bands
reach it; value = median over steps (time_pipeline's median,
eval.hpp:144-159).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK_GBS = 6650.0
WORDOPS_PER_CLK_SM = 32  # ALU: 64 LOP3/clk/SM at 2 LOP3 per word-op; XU: 16 POPC/clk/SM at 0.5 per word-op
WORKLOADS_CLI = ["c1", "c2", "c3", "c4", "c5", "c2rgb"]


def env_int(k, d):
    return int(os.environ.get(k, d))


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region.

    NVML in-process every 5 ms (the device found by its PCI bus id, so
    CUDA_VISIBLE_DEVICES remapping does not matter); `nvidia-smi` every 0.2 s
    when NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []  # (sm_mhz, max_mhz, {reason names})
        self.source = "nvidia-smi"
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            props = torch.cuda.get_device_properties(gpu)
            bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
            self._h = nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
            self._bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                          nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
            self._max = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._nvml = nv
            self.source = "nvml"
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        self.samples.append((float(sm), float(self._max),
                             {n for n, bit in zip(self.NAMES, self._bits) if r & bit}))

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        f = [x.strip() for x in out.split(",")]
        if len(f) >= 6 and f[0].replace(".", "").isdigit():
            self.samples.append((float(f[0]), float(f[1]) if f[1].replace(".", "").isdigit() else None,
                                 {n for n, v in zip(self.NAMES, f[2:6]) if v.lower() == "active"}))

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample_nvml() if self._nvml else self._sample_smi()
            except Exception:
                pass
            self._stop.wait(0.005 if self._nvml else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        mx = [s[1] for s in self.samples if s[1]]
        reasons = sorted(set().union(*(s[2] for s in self.samples)))
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples), "source": self.source}


def k3_tc_geometry(W: int, rows: int, D: int, nbits: int = 4096, masked: bool = True) -> dict:
    """Work of one k_cost_wta_tc launch (both directions), mirroring its host
    launch (bsm_kernels.cu wta_device_tc) and kern_cost_tc.cuh: 128-pixel tiles,
    d-blocks of <= 256, ncols accumulator columns, stages of 8 u32 words."""
    Wq = (W + 3) // 4 * 4
    tiles = (rows * Wq + 127) // 128
    ndd = (D + 255) // 256
    Dc = D if ndd == 1 else ((D + ndd - 1) // ndd + 3) // 4 * 4
    ncols = (128 + ((Dc + 2) & ~3) + 31) // 32 * 32
    NW = 2 * ((nbits + 63) // 64)
    nst = (NW + 7) // 8
    items = tiles * ndd * 2
    issued = 2.0 * items * 128 * ncols * nst * 8 * 32
    operand = (128 + ncols) * 8 * 16 * 2  # A + B rows x 8 words x 16 B, written and read
    raw = ((2 if masked else 1) * 8 * 128 * 4 + 8 * ncols * 4) * 2  # TMA-staged words, written and read
    return {"ncols": ncols, "items": items, "issued_flops": issued, "smem_bytes": float(items) * nst * (operand + raw)}


def in_bounds_evals(W, H, D):
    """Evaluations the reference performs per direction (matcher.hpp:100 skips x-d < 0)."""
    Dc = min(D, W)
    return H * (W * Dc - Dc * (Dc - 1) // 2)


# ---------------------------------------------------------------------------
# CPU legs: the reference compiled in place (oracle/_ref); inputs come from the
# generator compiled into that same library, so no product library is loaded.
def cpu_info() -> dict:
    model, mhz = None, []
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name") and model is None:
                    model = ln.split(":", 1)[1].strip()
                elif ln.startswith("cpu MHz"):
                    mhz.append(float(ln.split(":", 1)[1]))
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count() or 1
    return {"nproc": usable, "cpu_count": os.cpu_count(), "model": model,
            "mhz_median": statistics.median(mhz) if mhz else None}


def ref_inputs(ref, key: str, index: int = 0):
    from paper_1402_2020_b200.synth import workload_pair_with
    return workload_pair_with(ref.synth_pair, key, index)


def ref_band(ref, pairs_arr, left, right, y0, y1, d_max, threads):
    """run_pipeline of rows [y0, y1) as their own image; (seconds, W*rows*D)."""
    L = np.ascontiguousarray(left[y0:y1])
    R = np.ascontiguousarray(right[y0:y1])
    out = ref.pipeline(L, R, pairs_arr, 26, d_max, threads=threads, channels=3 if L.ndim == 3 else 1)
    return out["seconds"], L.shape[1] * (y1 - y0) * d_max


def run_reference(args):
    """--impl reference: the reference's own CPU implementation, rank 0 only."""
    if env_int("RANK", 0) != 0:
        return 0
    import oracle
    from paper_1402_2020_b200.synth import WORKLOADS
    w = WORKLOADS[args.workload]
    info = cpu_info()
    threads = info["nproc"]
    ref = oracle.Reference()
    pairs_arr = ref.generate_pattern(4096, 26, 4.0, 42)
    left, right = ref_inputs(ref, args.workload, 0)
    H = left.shape[0]
    if args.warmup > 0:  # page in the library and the thread pool on a small band
        ref_band(ref, pairs_arr, left, right, 0, min(8, H), w.d_max, threads)
    steps = max(1, args.steps)
    # consecutive bands walk down the frame (wrapping at the bottom); a band
    # holds at least 8 rows per thread so the reference's row-parallel
    # parallel_for (parallel.hpp:15-46) is balanced
    rows = min(H, max(-(-H // steps), 8 * threads))
    secs, evals, tput, covered = [], [], [], set()
    for i in range(steps):
        y0 = (i * rows) % H
        y1 = min(H, y0 + rows)
        s, e = ref_band(ref, pairs_arr, left, right, y0, y1, w.d_max, threads)
        secs.append(s)
        evals.append(e)
        tput.append(e / s / 1e6)
        covered.update(range(y0, y1))
    value = statistics.median(tput)
    frame = sum(evals) / sum(secs) / 1e6
    sample = (f"pair 0 of {w.name} ({w.width}x{H}, D={w.d_max}): {steps} consecutive bands of up to {rows} rows, "
              f"one per step, each run through run_pipeline as its own image ({len(covered)} of {H} rows "
              f"covered); {os.path.basename(ref.path)}, {threads} threads")
    line = {
        "impl": "reference", "metric": "Mdisp-evals/s", "value": value, "unit": "Mdisp-evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(secs) * 1e3, "higher_is_better": True,
        "scaling": "strong" if (w.pairs > 1 or args.workload == "c5") else "weak", "vs_baseline": None,
        "dtype": "u64 popcount / f64 votes",
        "data": ("synthetic colour views (synth.colour_pair)" if args.workload.endswith("rgb")
                 else "synthetic (BASELINE.json generator, SURVEY.md 8(d))"),
        "config": {"workload": w.name, "width": w.width, "height": w.height, "d_max": w.d_max, "n": 4096,
                   "pairs": w.pairs, "sample": "row bands of pair 0 tiling the frame, one per step",
                   "same_config": True},
        "cpu_baseline": {"value": value, "unit": "Mdisp-evals/s", "cores": threads, "kind": "reference",
                         "sample": sample, "whole_frame_value": frame, "cpu": info,
                         "statistic": "median over steps (eval.hpp:144-159 time_pipeline)"},
        "e2e": {"value": value, "unit": "Mdisp-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_leg(args, w, pairs_arr):
    """Bounded sample for the GPU arm's line (rank 0, N = 1): median of
    `--ref-repeats` runs of a `--ref-rows` band of pair 0 on all host threads,
    plus one run on one thread (the paper's protocol)."""
    import oracle
    info = cpu_info()
    threads = info["nproc"]
    ref = oracle.Reference()
    left, right = ref_inputs(ref, args.workload, 0)
    H = left.shape[0]
    rows = min(args.ref_rows or 8 * threads, H)
    y0 = (H - rows) // 2
    ref_band(ref, pairs_arr, left, right, y0, y0 + min(8, rows), w.d_max, threads)  # warm-up
    tp = []
    for _ in range(max(1, args.ref_repeats)):
        s, e = ref_band(ref, pairs_arr, left, right, y0, y0 + rows, w.d_max, threads)
        tp.append(e / s / 1e6)
    r1 = max(2, rows // 16)
    s1, e1 = ref_band(ref, pairs_arr, left, right, y0, y0 + r1, w.d_max, 1)
    return {"value": statistics.median(tp), "unit": "Mdisp-evals/s", "cores": threads, "kind": "reference",
            "sample": f"median of {len(tp)} runs of rows [{y0}, {y0 + rows}) x {w.width} x D={w.d_max} of pair 0, "
                      f"{os.path.basename(ref.path)}",
            "cpu": info, "single_thread": {"value": e1 / s1 / 1e6, "cores": 1,
                                           "sample": f"{r1} rows x {w.width} x D={w.d_max}"}}


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=WORKLOADS_CLI)
    ap.add_argument("--pairs", type=int, default=0, help="batch size override (c4; default: the config's 64)")
    ap.add_argument("--ref-rows", type=int, default=0, help="cpu_baseline band rows (0: 8 per host thread)")
    ap.add_argument("--ref-repeats", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="value loop only (for ncu)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import ctypes as C

    import torch
    import torch.distributed as dist

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    # ---- cold start: context + pattern + first pipeline (tables built lazily) ----
    t_cold = time.perf_counter()
    import paper_1402_2020_b200 as bsm
    from paper_1402_2020_b200._lib import bsm_maps, bsm_params, check, lib
    from paper_1402_2020_b200.dist import band_rows, shard_units
    from paper_1402_2020_b200.synth import WORKLOADS, workload_pair
    t_import = time.perf_counter()
    ctx = bsm.Context(local)
    t_ctx = time.perf_counter()
    w = WORKLOADS[args.workload]
    W, H, D = w.width, w.height, w.d_max
    cfg = bsm.BsmConfig(d_max=D)
    pattern = bsm.generate_pattern(cfg=cfg)
    ctx.set_pattern(pattern)
    t_pat = time.perf_counter()
    p = bsm_params(D, cfg.lambda_c, cfg.lambda_e, cfg.lr_tolerance, cfg.vote_radius)

    colour = args.workload.endswith("rgb")
    bands = args.workload == "c5" and world > 1
    n_total = (args.pairs or w.pairs) if w.pairs > 1 else 1
    batch = w.pairs > 1
    mine = list(shard_units(n_total, world, rank)) if batch else [0]
    views = [workload_pair(args.workload, index=i) for i in mine]
    px_view = W * H * (3 if colour else 1)
    d_l = [torch.from_numpy(l).to(dev) for l, _ in views]
    d_r = [torch.from_numpy(r).to(dev) for _, r in views]
    d_od = [torch.empty((H, W), dtype=torch.float32, device=dev) for _ in views]
    d_ov = [torch.empty((H, W), dtype=torch.uint8, device=dev) for _ in views]
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    vp = lambda ts: (C.c_void_p * max(1, len(ts)))(*[t.data_ptr() for t in ts])
    dl_arr, dr_arr, od_arr, ov_arr = vp(d_l), vp(d_r), vp(d_od), vp(d_ov)

    # first pipeline call (cold): the refine weight table and the other lazily
    # built device tables are created here
    t0 = time.perf_counter()
    fn_dev = lib().bsm_pipeline_rgb_device if colour else lib().bsm_pipeline_u8_device
    check(fn_dev(ctx.handle, C.c_void_p(d_l[0].data_ptr()), C.c_void_p(d_r[0].data_ptr()), W, H, C.byref(p), 0))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    check(fn_dev(ctx.handle, C.c_void_p(d_l[0].data_ptr()), C.c_void_p(d_r[0].data_ptr()), W, H, C.byref(p), 0))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cold = {"import_ms": (t_import - t_cold) * 1e3, "ctx_create_ms": (t_ctx - t_import) * 1e3,
            "set_pattern_ms": (t_pat - t_ctx) * 1e3, "first_pipeline_ms": (t1 - t0) * 1e3,
            "warm_pipeline_ms": (t2 - t1) * 1e3,
            "total_to_first_result_ms": (t1 - t_cold) * 1e3 - (t0 - t_pat) * 1e3}

    if bands:
        y0, y1 = band_rows(H, world, rank)
        rows_max = -(-H // world)
        band_d = torch.zeros((rows_max, W), dtype=torch.float32, device=dev)
        band_v = torch.zeros((rows_max, W), dtype=torch.uint8, device=dev)
        all_d = [torch.empty_like(band_d) for _ in range(world)]
        all_v = [torch.empty_like(band_v) for _ in range(world)]

    def step_device():
        if batch:
            check(lib().bsm_pipeline_batch_u8_device(ctx.handle, len(mine), dl_arr, dr_arr, W, H, C.byref(p),
                                                     od_arr, ov_arr))
            return
        if not bands:
            check(fn_dev(ctx.handle, C.c_void_p(d_l[0].data_ptr()), C.c_void_p(d_r[0].data_ptr()), W, H,
                         C.byref(p), 0))
            return
        check(lib().bsm_pipeline_band_u8_device(ctx.handle, C.c_void_p(d_l[0].data_ptr()),
                                                C.c_void_p(d_r[0].data_ptr()), W, H, y0, y1, C.byref(p)))
        check(lib().bsm_copy_result_device(ctx.handle, C.c_void_p(band_d.data_ptr()), C.c_void_p(band_v.data_ptr())))
        with torch.cuda.stream(stream):  # stream-ordered after the band kernels
            dist.all_gather(all_d, band_d)
            dist.all_gather(all_v, band_v)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    # ---- warm-up ----
    for _ in range(max(args.warmup, 1)):
        step_device()
    barrier()

    # ---- timed region: device-resident value ----
    evs = []
    launches = 0
    with ClockSampler(local) as clocks:
        barrier()
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)  # evict L2 between steps (outside the events)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step_device()
                launches += ctx.last_launch_count()
                e1.record(stream)
            evs.append((e0, e1))
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = float(sum(step_ms))
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    if batch:
        units_step = W * H * D * n_total
    elif bands:
        units_step = W * H * D
    else:
        units_step = W * H * D * world
    value = units_step * args.steps / (total_ms * 1e-3) / 1e6

    line = {
        "metric": "Mdisp-evals/s", "value": value, "unit": "Mdisp-evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if (batch or bands) else "weak", "vs_baseline": None,
        "dtype": "e2m1 (fp4) MMA with exact fp32 accumulation / u8 ranks / f64 votes",
        "data": ("synthetic colour views (synth.colour_pair: configs[0] scene, three tone curves + noise)" if colour
                 else "synthetic (BASELINE.json generator, SURVEY.md 8(d))"),
        "config": {"workload": w.name, "width": W, "height": H, "d_max": D, "n": 4096,
                   "pairs_per_step": n_total if batch else (1 if bands else world),
                   "pairs_per_rank": len(mine) if batch else 1,
                   "parallelism": (f"pairs sharded {n_total}/{world} per rank (no data-path collective)" if batch
                                   else (f"row bands x{world} + NCCL all-gather" if bands
                                         else (f"replicas x{world}" if world > 1 else "1 pair"))),
                   "l2": "256 MiB flush before every step (outside events); per-pair working set 2-9 GB >> L2"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if args.profile_only:
        if rank == 0:
            print(json.dumps(line), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- e2e through the public C ABI with pinned host buffers ----
    h_l = [torch.from_numpy(l).pin_memory() for l, _ in views]
    h_r = [torch.from_numpy(r).pin_memory() for _, r in views]
    h_d = [torch.empty((H, W), dtype=torch.float32).pin_memory() for _ in views]
    h_v = [torch.empty((H, W), dtype=torch.uint8).pin_memory() for _ in views]
    hl_arr, hr_arr, hd_arr, hv_arr = vp(h_l), vp(h_r), vp(h_d), vp(h_v)
    if bands:
        h_all_d = torch.empty((world * rows_max, W), dtype=torch.float32).pin_memory()
        h_all_v = torch.empty((world * rows_max, W), dtype=torch.uint8).pin_memory()
    maps = bsm_maps(h_d[0].data_ptr(), h_v[0].data_ptr(), None, None, None, None, None)

    def step_e2e():
        if batch:
            check(lib().bsm_pipeline_batch_u8(ctx.handle, len(mine), hl_arr, hr_arr, W, H, C.byref(p), hd_arr,
                                              hv_arr))
            return
        if not bands:
            fn = lib().bsm_pipeline_rgb if colour else lib().bsm_pipeline_u8
            check(fn(ctx.handle, C.c_void_p(h_l[0].data_ptr()), C.c_void_p(h_r[0].data_ptr()), W, H, C.byref(p), 0,
                     C.byref(maps)))
            return
        with torch.cuda.stream(stream):
            d_l[0].copy_(h_l[0], non_blocking=True)
            d_r[0].copy_(h_r[0], non_blocking=True)
        step_device()
        with torch.cuda.stream(stream):
            h_all_d.copy_(torch.cat(all_d), non_blocking=True)
            h_all_v.copy_(torch.cat(all_v), non_blocking=True)
        stream.synchronize()

    step_e2e()
    barrier()
    e2e_ms, e2e_wall = [], []
    for _ in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tw = time.perf_counter()
        step_e2e()
        e1.record(stream)
        e1.synchronize()
        e2e_wall.append((time.perf_counter() - tw) * 1e3)
        e2e_ms.append(e0.elapsed_time(e1))
    barrier()
    te = torch.tensor([float(sum(e2e_ms))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = units_step * args.steps / (float(te.item()) * 1e-3) / 1e6
    if batch:
        h2d, d2h = 2 * px_view * len(mine), 5 * W * H * len(mine)
    elif bands:
        h2d, d2h = 2 * px_view, 5 * world * rows_max * W
    else:
        h2d, d2h = 2 * px_view, 5 * W * H
    line["e2e"] = {"value": e2e_value, "unit": "Mdisp-evals/s", "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h, "ms_per_step": float(te.item()) / args.steps,
                   "host_wall_ms_per_step": float(np.mean(e2e_wall)),
                   "call": ("bsm_pipeline_batch_u8" if batch else ("bsm_pipeline_band_u8_device + NCCL all-gather"
                                                                   if bands else
                                                                   ("bsm_pipeline_rgb" if colour else
                                                                    "bsm_pipeline_u8")))}

    # ---- per-stage device time of one pair (events on the library's stream) ----
    ctx.set_profiling(True)
    prof = {}
    for _ in range(max(3, min(args.steps, 8))):
        flush.fill_(1)
        torch.cuda.synchronize()
        if bands:
            check(lib().bsm_pipeline_band_u8_device(ctx.handle, C.c_void_p(d_l[0].data_ptr()),
                                                    C.c_void_p(d_r[0].data_ptr()), W, H, y0, y1, C.byref(p)))
        else:
            check(fn_dev(ctx.handle, C.c_void_p(d_l[0].data_ptr()), C.c_void_p(d_r[0].data_ptr()), W, H,
                         C.byref(p), 0))
        for k, v in ctx.last_timings().items():
            prof.setdefault(k, []).append(v)
    ctx.set_profiling(False)
    prof_ms = {k: float(np.median(v)) for k, v in prof.items() if np.median(v) > 0}  # median: robust to one slow run
    mma_peak = ctx.measure_mma_peak()  # live dense FP4 tensor rate, flop/s

    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    peaks = json.load(open(MEASURED_PEAKS)) if os.path.exists(MEASURED_PEAKS) else {}
    clk = line["clocks"].get("sm_max_mhz") or peaks.get("sm_max_mhz") or 1965.0
    pipe_peak = WORDOPS_PER_CLK_SM * sms * clk * 1e6  # nominal word-ops/s of the popcount formulation
    rows_c = (min(H, y1 + cfg.vote_radius) - max(0, y0 - cfg.vote_radius)) if bands else H
    evals_dir = in_bounds_evals(W, rows_c, D)
    wta_ms = prof_ms.get("wta", 0.0) + prof_ms.get("wta_left", 0.0) + prof_ms.get("wta_right", 0.0)
    sec = wta_ms * 1e-3
    k3 = k3_tc_geometry(W, rows_c, D, nbits=4096)
    alg_flops = 2.0 * 2 * evals_dir * 4096  # one MAC per descriptor bit per in-bounds (x, y, d, direction)
    hbm_peak = peaks.get("hbm_gbs", HBM_FALLBACK_GBS)
    alg_bytes = 2 * W * rows_c * (3 * 4096 // 8 + 4)  # per direction: ref desc + ref mask + other desc, + key
    traffic = mask_traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        traffic = tj.get("k_cost_wta_tc", {}).get(args.workload)
        mask_traffic = tj.get("k_mask", {}).get(args.workload)
    smem_peak = 128 * sms * clk * 1e6  # B/s: 128 B/clk/SM
    line["roofline_cost"] = {
        "bound": "tensor (tcgen05 kind::mxf4, dense FP4)",
        "kernel": "k_cost_wta_tc (masked Hamming as a banded FP4 MMA + fused WTA, both directions)",
        "achieved": alg_flops / sec / 1e12, "peak": mma_peak / 1e12, "unit": "TFLOP/s",
        "frac": alg_flops / sec / mma_peak, "traffic": traffic,
        "peak_source": "live: kind::mxf4 M128 N256 K64 MMAs issued back to back, one CTA per SM "
                       "(bsm_measure_mma_peak); nominal dense FP4 9000 TFLOP/s",
        "unit_def": "algorithmic flop = 2 per descriptor bit per in-bounds (x, y, d, direction): "
                    "popc((a^b)&m) = popc(a&m) + sum m(1-2a)b",
        "kernel_ms": wta_ms, "alg_flops": alg_flops,
        "issued_flops": k3["issued_flops"], "mma_busy_frac": k3["issued_flops"] / sec / mma_peak,
        "band_efficiency": alg_flops / k3["issued_flops"],
        # what binds it: every operand byte is written by the producers and read by the
        # tensor core through shared memory, and the packed words are staged there by TMA
        "smem": {"bytes": k3["smem_bytes"], "achieved_gbs": k3["smem_bytes"] / sec / 1e9,
                 "peak_gbs": smem_peak / 1e9, "frac": k3["smem_bytes"] / sec / smem_peak,
                 "peak_source": f"128 B/clk/SM x {sms} SMs x {clk:.0f} MHz"},
        "int_pipe_equiv": {"achieved_gwordops": 2 * evals_dir * 128 / sec / 1e9,
                           "int_pipe_peak_gwordops": pipe_peak / 1e9,
                           "x_int_pipe_roofline": 2 * evals_dir * 128 / sec / pipe_peak,
                           "note": "the same work as u32 (a^b)&m + popcount word-ops against the nominal "
                                   "ALU+XU bound of the popcount formulation (32 word-ops/clk/SM)"},
        "hbm_achieved_gbs": alg_bytes / sec / 1e9, "hbm_peak_gbs": hbm_peak,
        "hbm_frac": alg_bytes / sec / 1e9 / hbm_peak,
    }
    mask_ms = prof_ms.get("mask", 0.0)
    if mask_ms > 0 and not colour:
        # K2: 2 rank gathers per pair and pixel; the ranks are u8, so one 32-bit
        # shared-memory gather can serve four pixels (k_mask_q does):
        # n / 64 conflict-free wavefronts per pixel is the gather floor of any
        # table-driven implementation; the LSU serves 1 per clk per SM
        # (the library's choice for n = 4096: k_mask_q unless BSM_MASK_VARIANT selects k_mask4)
        mask_kernel = "k_mask4" if int(os.environ.get("BSM_MASK_VARIANT", "0")) & 3 else "k_mask_q"
        wf = 2 * W * rows_c * (4096 // 64)  # both views
        wf_peak = sms * clk * 1e6
        line["roofline_mask"] = {"bound": "smem (L1 shared-memory wavefronts of the rank gathers)",
                                 "kernel": f"{mask_kernel} (both views)",
                                 "achieved": wf * 128 / (mask_ms * 1e-3) / 1e9, "peak": smem_peak / 1e9,
                                 "unit": "GB/s", "frac": wf / (mask_ms * 1e-3) / wf_peak, "traffic": mask_traffic,
                                 "peak_source": f"1 wavefront (128 B) / clk / SM x {sms} SMs x {clk:.0f} MHz",
                                 "kernel_ms": mask_ms, "wavefronts": wf,
                                 # HBM side (both views): one image byte in, n/8 mask bytes out per pixel
                                 "hbm_achieved_gbs": 2 * W * rows_c * (1 + 4096 // 8) / (mask_ms * 1e-3) / 1e9,
                                 "hbm_peak_gbs": hbm_peak,
                                 "hbm_frac": 2 * W * rows_c * (1 + 4096 // 8) / (mask_ms * 1e-3) / 1e9 / hbm_peak,
                                 "unit_def": "n/64 = 64 rank-gather wavefronts per pixel (2 gathers per pair, four "
                                             "pixels' u8 ranks per u32), 128 B each",
                                 "note": "the kernel is instruction-issue-bound (~69% issue slots busy, L1 58%, "
                                         "ncu: profiles/r02_ncu_kernels_c4.txt): bit-plane transposes and the "
                                         "select, not the gathers, set its time"}
    # the contract's `roofline` is the dominant kernel of the step (by measured stage time)
    cands = [line["roofline_cost"]] + ([line["roofline_mask"]] if "roofline_mask" in line else [])
    line["roofline"] = dict(max(cands, key=lambda r: r["kernel_ms"]))
    line["roofline"]["step_share"] = line["roofline"]["kernel_ms"] / max(sum(prof_ms.values()), 1e-9)
    line["stage_ms"] = prof_ms
    line["cold_start"] = cold
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline_leg(args, w, pattern.pairs)
        except Exception as ex:  # the checker is optional on a box without it
            line["cpu_baseline"] = {"value": None, "error": str(ex)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
