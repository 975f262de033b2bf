#!/usr/bin/env python
"""Benchmark of the Binary Stereo Matching hot path on B200.

metric: Mdisp-evals/s = W*H*D per second (BASELINE.json), whole job.

Default workload: BASELINE.json configs[1] (1392x1104, D=240, the largest
single-pair config quoted for 1 GPU).  One step = one full run_pipeline of one
stereo pair: descriptors + masks of both views, masked WTA in both
directions, left/right check, voting refinement.  N > 1 (torchrun): every rank
matches its own pair (independent units, weak scaling, no data-path
collective -- the batch partition of configs[3]).

  value   device-resident inputs, CUDA events on the library's stream per step
          (L2 flushed by a 256 MiB write before each step, outside the events)
  e2e     the public C-ABI call bsm_pipeline_u8 with pinned HOST buffers: the
          H2D of both views and the D2H of the refined map (float + valid) are
          inside the timed region
  roofline  the dominant kernel (fused masked-Hamming cost + WTA) against the
          measured POPC word-op rate of this GPU (it is POPC-issue bound, not
          HBM bound -- see DESIGN.md); hbm_frac beside it
  cpu_baseline  the reference library compiled in place (oracle/_ref), all
          host threads, on a bounded row band of the same workload

--impl reference: the reference CPU implementation alone (rank 0), same
metric, on a bounded row band per step.
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


def in_bounds_evals(W, H, D):
    """Evaluations the reference performs per direction (matcher.hpp:100 skips x-d < 0)."""
    Dc = min(D, W)
    return H * (W * Dc - Dc * (Dc - 1) // 2)


def cpu_reference_sample(workload, rows, threads, pairs_arr):
    """Reference pipeline (oracle/_ref) on a row band of the workload's pair."""
    import oracle
    from paper_1402_2020_b200.synth import workload_pair
    ref = oracle.Reference()
    left, right = workload_pair(workload)
    y0 = (left.shape[0] - rows) // 2
    L = np.ascontiguousarray(left[y0:y0 + rows])
    R = np.ascontiguousarray(right[y0:y0 + rows])
    from paper_1402_2020_b200.synth import WORKLOADS
    w = WORKLOADS[workload]
    out = ref.pipeline(L, R, pairs_arr, 26, w.d_max, threads=threads, channels=3 if L.ndim == 3 else 1)
    return out["seconds"], L.shape[1] * rows * w.d_max, os.path.basename(ref.path)


def run_reference(args):
    """--impl reference: the reference's own CPU implementation, rank 0 only."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    import oracle
    from paper_1402_2020_b200.synth import WORKLOADS
    w = WORKLOADS[args.workload]
    threads = os.cpu_count() or 1
    pairs_arr = oracle.Reference().generate_pattern(4096, 26, 4.0, 42)
    rows = args.ref_rows
    for _ in range(args.warmup if args.warmup <= 1 else 1):
        cpu_reference_sample(args.workload, max(8, rows // 4), threads, pairs_arr)
    secs, evals = 0.0, 0
    for _ in range(args.steps):
        s, e, lib = cpu_reference_sample(args.workload, rows, threads, pairs_arr)
        secs += s
        evals += e
    v = evals / secs / 1e6
    line = {
        "impl": "reference", "metric": "Mdisp-evals/s", "value": v, "unit": "Mdisp-evals/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32 popcount / f64 votes",
        "data": ("synthetic colour views (synth.colour_pair)" if args.workload.endswith("rgb")
                 else "synthetic (BASELINE.json generator, SURVEY.md 8(d))"),
        "config": {"workload": w.name, "width": w.width, "height": w.height, "d_max": w.d_max, "n": 4096,
                   "sample": f"{rows}-row band per step"},
        "cpu_baseline": {"value": v, "unit": "Mdisp-evals/s", "cores": threads, "kind": "reference",
                         "sample": f"{rows} rows x {w.width} x D={w.d_max} per step, {lib}"},
        "e2e": {"value": v, "unit": "Mdisp-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5", "c2rgb"])
    ap.add_argument("--ref-rows", type=int, default=48)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="few steps, no CPU leg (for ncu)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_1402_2020_b200 as bsm
    from paper_1402_2020_b200.synth import WORKLOADS, workload_pair

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = WORKLOADS[args.workload]
    W, H, D = w.width, w.height, w.d_max

    ctx = bsm.Context(local)
    cfg = bsm.BsmConfig(d_max=D)
    pattern = bsm.generate_pattern(cfg=cfg)
    ctx.set_pattern(pattern)
    # Partition: configs[4] (c5, one frame) -> contiguous row
    # bands with a vote-radius halo + one NCCL all-gather of the refined bands
    # (strong scaling); every other workload -> rank r matches pair index r of
    # the workload's seed sequence (independent units, weak scaling).
    bands = args.workload == "c5" and world > 1
    colour = args.workload.endswith("rgb")  # interleaved RGB views (colour path)
    left, right = workload_pair(args.workload, index=0 if bands else rank)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    d_left = torch.from_numpy(left).to(dev)
    d_right = torch.from_numpy(right).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    from paper_1402_2020_b200._lib import check, lib, bsm_params
    import ctypes as C
    p = bsm_params(D, cfg.lambda_c, cfg.lambda_e, cfg.lr_tolerance, cfg.vote_radius)

    if bands:
        from paper_1402_2020_b200.dist import band_rows
        y0, y1 = band_rows(H, world, rank)
        rows_max = -(-H // world)
        band_d = torch.zeros((rows_max, W), dtype=torch.float32, device=dev)
        band_v = torch.zeros((rows_max, W), dtype=torch.uint8, device=dev)
        all_d = [torch.empty_like(band_d) for _ in range(world)]
        all_v = [torch.empty_like(band_v) for _ in range(world)]

    def step_device():
        if colour:
            check(lib().bsm_pipeline_rgb_device(ctx.handle, C.c_void_p(d_left.data_ptr()),
                                                C.c_void_p(d_right.data_ptr()), W, H, C.byref(p), 0))
            return
        if not bands:
            check(lib().bsm_pipeline_u8_device(ctx.handle, C.c_void_p(d_left.data_ptr()),
                                               C.c_void_p(d_right.data_ptr()), W, H, C.byref(p), 0))
            return
        check(lib().bsm_pipeline_band_u8_device(ctx.handle, C.c_void_p(d_left.data_ptr()),
                                                C.c_void_p(d_right.data_ptr()), W, H, y0, y1, C.byref(p)))
        check(lib().bsm_copy_result_device(ctx.handle, C.c_void_p(band_d.data_ptr()), C.c_void_p(band_v.data_ptr())))
        with torch.cuda.stream(stream):  # stream-ordered after the band kernels
            dist.all_gather(all_d, band_d)
            dist.all_gather(all_v, band_v)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    # ---- warm-up (also builds the refine weight table once) ----
    for _ in range(max(args.warmup, 1)):
        step_device()
    barrier()

    # ---- timed region: device-resident value ----
    evs = []
    with ClockSampler(local) as clocks:
        barrier()
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)  # evict L2 between steps (outside the events)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step_device()
                e1.record(stream)
            evs.append((e0, e1))
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = float(sum(step_ms))
    launches = ctx.last_launch_count()
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    units = W * H * D * (1 if bands else world) * args.steps
    value = units / (total_ms * 1e-3) / 1e6

    # ---- e2e through the public C ABI with pinned host buffers ----
    h_left = torch.from_numpy(left).pin_memory()
    h_right = torch.from_numpy(right).pin_memory()
    h_rd = torch.empty((H, W), dtype=torch.float32).pin_memory()
    h_rv = torch.empty((H, W), dtype=torch.uint8).pin_memory()
    maps = bsm._lib.bsm_maps(h_rd.data_ptr(), h_rv.data_ptr(), None, None, None, None, None)

    if bands:
        h_all_d = torch.empty((world * rows_max, W), dtype=torch.float32).pin_memory()
        h_all_v = torch.empty((world * rows_max, W), dtype=torch.uint8).pin_memory()

    def step_e2e():
        if not bands:
            fn = lib().bsm_pipeline_rgb if colour else lib().bsm_pipeline_u8
            check(fn(ctx.handle, C.c_void_p(h_left.data_ptr()), C.c_void_p(h_right.data_ptr()),
                     W, H, C.byref(p), 0, C.byref(maps)))
            return
        with torch.cuda.stream(stream):
            d_left.copy_(h_left, non_blocking=True)
            d_right.copy_(h_right, non_blocking=True)
        step_device()
        with torch.cuda.stream(stream):
            h_all_d.copy_(torch.cat(all_d), non_blocking=True)
            h_all_v.copy_(torch.cat(all_v), non_blocking=True)
        stream.synchronize()

    step_e2e()
    barrier()
    e2e_ms = []
    for _ in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step_e2e()
        e1.record(stream)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    barrier()
    te = torch.tensor([float(sum(e2e_ms))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = units / (float(te.item()) * 1e-3) / 1e6

    # ---- per-kernel device time (events on the library's stream) ----
    ctx.set_profiling(True)
    prof = {}
    nprof = max(3, min(args.steps, 10))
    for _ in range(nprof):
        flush.fill_(1)
        torch.cuda.synchronize()
        step_device()
        for k, v in ctx.last_timings().items():
            prof.setdefault(k, []).append(v)
    ctx.set_profiling(False)
    prof_ms = {k: float(np.mean(v)) for k, v in prof.items() if np.mean(v) > 0}
    popc_peak, csa_peak = ctx.measure_word_peaks()  # word-ops/s, this GPU, live

    if bands:  # fields / WTA / check cover the band plus the vote-radius halo
        hr = min(H, y1 + cfg.vote_radius) - max(0, y0 - cfg.vote_radius)
        evals_dir = in_bounds_evals(W, hr, D)
    else:
        evals_dir = in_bounds_evals(W, H, D)
    wta_ms = (prof_ms.get("wta_left", 0) + prof_ms.get("wta_right", 0)) / 2
    achieved = evals_dir * (4096 // 32) / (wta_ms * 1e-3)  # u32 masked-xor-popcount word-ops / s
    peaks = json.load(open(MEASURED_PEAKS)) if os.path.exists(MEASURED_PEAKS) else {}
    hbm_peak = peaks.get("hbm_gbs", HBM_FALLBACK_GBS)
    alg_bytes = W * (hr if bands else H) * (3 * 4096 // 8 + 4)  # ref desc + ref mask + other desc, + key
    hbm_ach = alg_bytes / (wta_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(args.workload)

    line = {
        "metric": "Mdisp-evals/s", "value": value, "unit": "Mdisp-evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if bands else "weak", "vs_baseline": None,
        "dtype": "u32 popcount / f64 votes",
        "data": ("synthetic colour views (synth.colour_pair: configs[0] scene, three tone curves + noise)" if colour
                 else "synthetic (BASELINE.json generator, SURVEY.md 8(d))"),
        "config": {"workload": w.name, "width": W, "height": H, "d_max": D, "n": 4096,
                   "pairs_per_step": 1 if bands else world,
                   "parallelism": (f"row bands x{world} + NCCL all-gather" if bands
                                   else (f"pairs x{world}" if world > 1 else "1 pair")),
                   "l2": "256 MiB flush before every step (outside events); working set 3.2 GB >> L2"},
        "e2e": {"value": e2e_value, "unit": "Mdisp-evals/s", "h2d_bytes_per_step": 2 * W * H * (3 if colour else 1),
                "d2h_bytes_per_step": 5 * (world * rows_max if bands else H) * W,
                "ms_per_step": float(te.item()) / args.steps},
        "gpu_launches": launches * args.steps,
        "roofline": {"bound": "int-pipes (LOP3+POPC)",
                     "kernel": "k_cost_wta (fused masked Hamming + WTA, per direction)",
                     "achieved": achieved / 1e9, "peak": csa_peak / 1e9, "unit": "Gword-ops/s",
                     "frac": achieved / csa_peak, "traffic": traffic,
                     "peak_source": "live register-only microbenchmark of the kernel's carry-save instruction mix "
                                    "(2 words per 4 LOP3 + POPC + IMAD: ALU and POPC pipes balanced) on this GPU",
                     "popc_only_peak": popc_peak / 1e9, "frac_of_popc_only": achieved / popc_peak,
                     "kernel_ms": wta_ms, "alg_word_ops_per_launch": evals_dir * 128,
                     "hbm_achieved_gbs": hbm_ach, "hbm_peak_gbs": hbm_peak, "hbm_frac": hbm_ach / hbm_peak},
        "stage_ms": prof_ms,
        "clocks": clocks.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile_only:
        try:
            pairs_arr = pattern.pairs
            threads = os.cpu_count() or 1
            s, e, libname = cpu_reference_sample(args.workload, args.ref_rows, threads, pairs_arr)
            line["cpu_baseline"] = {"value": e / s / 1e6, "unit": "Mdisp-evals/s", "cores": threads,
                                    "kind": "reference",
                                    "sample": f"{args.ref_rows} rows x {W} x D={D} of the same pair, {libname}"}
            # the paper's protocol is one thread: a smaller band
            r1 = max(4, args.ref_rows // 8)
            s1, e1, _ = cpu_reference_sample(args.workload, r1, 1, pairs_arr)
            line["cpu_baseline"]["single_thread"] = {"value": e1 / s1 / 1e6, "cores": 1,
                                                     "sample": f"{r1} rows x {W} x D={D}"}
        except Exception as ex:  # the checker is optional on a box without it
            line["cpu_baseline"] = {"value": None, "error": str(ex)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
