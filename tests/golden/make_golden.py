"""Generate golden fixtures from the reference library compiled in place
(oracle/_ref) on the BASELINE synthetic workloads.

Run here (the reference sources only exist in this container):
    python tests/golden/make_golden.py c1 c3 c2 c5 c4:0-3 rgb:640x480:3:64
Writes tests/golden/<key>.json (sha256 of every map + summary stats) and, for
the small c1 / c3 workloads, the maps themselves as <key>_maps.npz.
`rgb:<W>x<H>:<seed>:<d_max>` is a colour pair (paper_1402_2020_b200.synth.colour_pair)
through the reference's colour path (RgbImage with r, g, b distinct).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1402_2020_b200.synth import WORKLOADS, colour_pair, workload_pair  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run(key: str, index: int, threads: int) -> None:
    w = WORKLOADS[key]
    ref = oracle.Reference()
    pairs = ref.generate_pattern(4096, 26, 4.0, 42)
    left, right = workload_pair(key, index)
    t0 = time.time()
    out = ref.pipeline(left, right, pairs, 26, w.d_max, threads=threads)
    dt = time.time() - t0
    tag = key if w.pairs == 1 else f"{key}_{index}"
    rec = {
        "workload": w.name, "index": index, "width": w.width, "height": w.height, "d_max": w.d_max,
        "seed": w.seed + index, "pattern": {"n": 4096, "S": 26, "spread": 4.0, "seed": 42},
        "inputs": {"left": sha(left), "right": sha(right)},
        "maps": {k: sha(v) for k, v in out.items() if k != "seconds" and k != "unmasked_d"},
        "checked_invalid_frac": float(1.0 - out["checked_v"].mean()),
        "refined_invalid_frac": float(1.0 - out["refined_v"].mean()),
        "ref_library": os.path.basename(ref.path), "ref_threads": threads, "ref_seconds": dt,
    }
    with open(os.path.join(HERE, f"{tag}.json"), "w") as f:
        json.dump(rec, f, indent=1)
    if key in ("c1", "c3"):
        np.savez_compressed(os.path.join(HERE, f"{tag}_maps.npz"),
                            **{k: (v.astype(np.uint16) if v.dtype == np.float32 else v)
                               for k, v in out.items() if k not in ("seconds", "unmasked_d")})
    print(tag, f"{dt:.1f}s", rec["checked_invalid_frac"], flush=True)


def run_rgb(spec: str, threads: int) -> None:
    size, seed, d_max = spec.split(":")
    W, H = (int(v) for v in size.split("x"))
    seed, d_max = int(seed), int(d_max)
    ref = oracle.Reference()
    pairs = ref.generate_pattern(4096, 26, 4.0, 42)
    left, right = colour_pair(H, W, seed=seed)
    t0 = time.time()
    out = ref.pipeline(left, right, pairs, 26, d_max, threads=threads, channels=3)
    dt = time.time() - t0
    tag = f"rgb_{W}x{H}_s{seed}"
    rec = {
        "workload": "colour_pair", "width": W, "height": H, "d_max": d_max, "seed": seed,
        "pattern": {"n": 4096, "S": 26, "spread": 4.0, "seed": 42},
        "inputs": {"left": sha(left), "right": sha(right)},
        "maps": {k: sha(v) for k, v in out.items() if k != "seconds" and k != "unmasked_d"},
        "checked_invalid_frac": float(1.0 - out["checked_v"].mean()),
        "refined_invalid_frac": float(1.0 - out["refined_v"].mean()),
        "ref_library": os.path.basename(ref.path), "ref_threads": threads, "ref_seconds": dt,
    }
    with open(os.path.join(HERE, f"{tag}.json"), "w") as f:
        json.dump(rec, f, indent=1)
    print(tag, f"{dt:.1f}s", rec["checked_invalid_frac"], flush=True)


if __name__ == "__main__":
    threads = int(os.environ.get("THREADS", os.cpu_count() or 1))
    for arg in sys.argv[1:]:
        if arg.startswith("rgb:"):
            run_rgb(arg[4:], threads)
        elif ":" in arg:
            key, rng = arg.split(":")
            a, b = (int(x) for x in rng.split("-"))
            for i in range(a, b + 1):
                run(key, i, threads)
        else:
            run(arg, 0, threads)
