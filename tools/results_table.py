"""Print the DESIGN.md §10 / BASELINE.md §5 result rows from an evidence run's
bench lines.

    python tools/results_table.py <tag>     # reads gpurun_out/<tag>_bench_<wl>.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ROWS = [("default", "**c4 64 × 1920×1080 D=192 (headline)**"), ("c1", "c1 450×375 D=60"),
        ("c2", "c2 1392×1104 D=240"), ("c3", "c3 640×480 D=64"), ("c5", "c5 4096×2160 D=256"),
        ("c2rgb", "c2rgb (colour)")]


def line(tag, wl):
    txt = open(os.path.join(ROOT, "gpurun_out", f"{tag}_bench_{wl}.json")).read().strip().splitlines()[-1]
    return json.loads(txt)


def main():
    tag = sys.argv[1]
    for wl, name in ROWS:
        d = line(tag, wl)
        pairs = d["config"].get("pairs_per_step", 1) or 1
        ms_pair = d["ms_per_step"] / pairs
        rc, rm, st = d["roofline_cost"], d.get("roofline_mask", {}), d["stage_ms"]
        mask = f"{rm['frac']:.3f}" if rm else "—"
        print(f"| {name} | {d['value']:,.0f} ({d['e2e']['value']:,.0f}) | {ms_pair:.2f} | {rc['frac']:.3f} "
              f"({rc['smem']['frac']:.3f}) | {mask} | {st['descriptor']:.2f} / {st['mask']:.2f} / "
              f"{st['wta']:.2f} / {st['refine']:.2f} |")
    for wl in ("reference", "reference_c2"):
        d = line(tag, wl)
        print(wl, f"{d['value']:.1f}")


if __name__ == "__main__":
    main()
