"""Command-line front end over the GPU pipeline.

Same subcommands, flags, output files and printed lines as the reference tool
(tools/bsm.cpp:93-246):

    python -m paper_1402_2020_b200 match LEFT RIGHT OUT [--stages] [--pattern P] [--emit-pattern P] ...
    python -m paper_1402_2020_b200 eval RESULT GT [--nonocc M] [--all M] [--disc M] [--threshold T]
    python -m paper_1402_2020_b200 sweep SCENE_DIR... [--n_values 512,1024] [--out CSV]
    python -m paper_1402_2020_b200 radiometric SET_DIR [--out CSV]
    python -m paper_1402_2020_b200 bench LEFT RIGHT [--runs K]

plus the shared config flags (--config, --n, --S, --spread, --seed, --d_max,
--lambda_c, --lambda_e, --lr_tolerance, --vote_radius, --gt_scale, --threads);
explicit flags override a --config file, which overrides the defaults.
"""
from __future__ import annotations

import argparse
import os
import sys
from typing import List, Optional

from . import BsmConfig, generate_pattern, run_pipeline, to_gray_lab
from . import evaluation as ev
from . import io as bio
from ._lib import BsmError

_CFG_FLAGS = [  # flag, attribute, type (tools/bsm.cpp:13-27)
    ("--n", "n", int), ("--S", "window", int), ("--spread", "spread", float), ("--seed", "seed", int),
    ("--d_max", "d_max", int), ("--lambda_c", "lambda_c", float), ("--lambda_e", "lambda_e", float),
    ("--lr_tolerance", "lr_tolerance", float), ("--vote_radius", "vote_radius", int),
    ("--gt_scale", "gt_scale", float), ("--threads", "threads", int),
]


def _add_config_flags(p: argparse.ArgumentParser) -> None:
    p.add_argument("--config", help="JSON config file; explicit flags override its values")
    for flag, attr, typ in _CFG_FLAGS:
        p.add_argument(flag, dest="cfg_" + attr, type=typ, default=None)


def _scan_config_path(argv: List[str]) -> Optional[str]:
    """The config file loads before flags apply (tools/bsm.cpp:29-38)."""
    for i, a in enumerate(argv):
        if a == "--config" and i + 1 < len(argv):
            return argv[i + 1]
        if a.startswith("--config="):
            return a[len("--config="):]
    return None


def _stage_path(out: str, stage: str) -> str:
    root, ext = os.path.splitext(out)
    return f"{root}.{stage}{ext}"


def _write_map(m, path: str, scale: float) -> None:
    if os.path.splitext(path)[1] == ".pfm":
        bio.save_disparity_pfm(m, path)
    else:
        bio.save_disparity(m, path, scale)


def _report(label: str, rep: ev.ErrorReport) -> None:
    print("%-8s %6.2f  (%d of %d pixels beyond %.2f)" % (label, rep.bad_pixel_rate, rep.bad, rep.counted,
                                                           rep.threshold))


def _mask(path: str):
    g, _ = to_gray_lab(bio.load_image(path))
    return g


def _lookup(name: str):
    for nm, d, s in bio.MIDDLEBURY_SCENES:
        if nm == name:
            return d, s
    return None


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="bsm", description="binary-descriptor stereo matcher (B200)",
                                 allow_abbrev=False)
    sub = ap.add_subparsers(dest="cmd", required=True)
    m = sub.add_parser("match", help="compute a left-reference disparity map", allow_abbrev=False)
    m.add_argument("left")
    m.add_argument("right")
    m.add_argument("out")
    m.add_argument("--stages", action="store_true", help="also write the per-stage maps")
    m.add_argument("--pattern", default="", help="reuse a saved sampling pattern")
    m.add_argument("--emit-pattern", dest="emit_pattern", default="", help="save the sampling pattern used")
    _add_config_flags(m)
    e = sub.add_parser("eval", help="bad-pixel rate of a map against ground truth", allow_abbrev=False)
    e.add_argument("result")
    e.add_argument("gt")
    e.add_argument("--nonocc", default="")
    e.add_argument("--all", dest="all_mask", default="")
    e.add_argument("--disc", default="")
    e.add_argument("--threshold", type=float, default=1.0)
    _add_config_flags(e)
    s = sub.add_parser("sweep", help="accuracy and wall time across descriptor lengths", allow_abbrev=False)
    s.add_argument("scenes", nargs="+")
    s.add_argument("--n_values", default="512,1024,2048,4096")
    s.add_argument("--out", default="sweep.csv")
    s.add_argument("--threshold", type=float, default=1.0)
    _add_config_flags(s)
    r = sub.add_parser("radiometric", help="3x3 exposure-combination error grid", allow_abbrev=False)
    r.add_argument("set")
    r.add_argument("--out", default="radiometric.csv")
    r.add_argument("--threshold", type=float, default=1.0)
    _add_config_flags(r)
    b = sub.add_parser("bench", help="median wall time of the full pipeline", allow_abbrev=False)
    b.add_argument("left")
    b.add_argument("right")
    b.add_argument("--runs", type=int, default=3)
    _add_config_flags(b)
    return ap


def main(argv: Optional[List[str]] = None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    try:
        path = _scan_config_path(argv)
        cfg = bio.load_config(path) if path else BsmConfig()
    except BsmError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    try:
        a = _parser().parse_args(argv)
    except SystemExit as e:
        return int(e.code or 0)
    for _, attr, _t in _CFG_FLAGS:
        v = getattr(a, "cfg_" + attr)
        if v is not None:
            setattr(cfg, attr, v)
    try:
        if a.cmd == "match":
            left, right = bio.load_image(a.left), bio.load_image(a.right)
            cfg.validate()
            pattern = bio.load_pattern(a.pattern) if a.pattern else generate_pattern(cfg=cfg)
            res = run_pipeline(left, right, cfg, pattern, want_unmasked=a.stages)
            _write_map(res.refined, a.out, cfg.gt_scale)
            bio.save_config(cfg, a.out + ".config.json")
            if a.stages:
                _write_map(res.unmasked, _stage_path(a.out, "unmasked"), cfg.gt_scale)
                _write_map(res.left_wta, _stage_path(a.out, "masked"), cfg.gt_scale)
                _write_map(res.refined, _stage_path(a.out, "refined"), cfg.gt_scale)
            if a.emit_pattern:
                bio.save_pattern(pattern, a.emit_pattern)
        elif a.cmd == "eval":
            result = bio.load_gt_disparity(a.result, cfg.gt_scale)
            gt = bio.load_gt_disparity(a.gt, cfg.gt_scale)
            if not (a.nonocc or a.all_mask or a.disc):
                _report("all", ev.bad_pixel_rate(result, gt, None, a.threshold))
            else:
                for label, p in (("nonocc", a.nonocc), ("all", a.all_mask), ("disc", a.disc)):
                    if p:
                        _report(label, ev.bad_pixel_rate(result, gt, _mask(p), a.threshold))
        elif a.cmd == "sweep":
            n_values = [int(t) for t in a.n_values.split(",") if t.strip()]
            sets = []
            for d in a.scenes:
                name = os.path.basename(os.path.normpath(d))
                known = _lookup(name)
                dm = cfg.d_max if cfg.d_max > 0 else (known[0] if known else 0)
                if dm < 1:
                    raise bio.InvalidArgument(f"sweep: {d} is not a known scene, pass --d_max")
                sets.append(bio.load_stereo_dataset(d, name, dm, known[1] if known else cfg.gt_scale))
            scenes = [ev.SweepScene(s.left, s.right, s.gt, s.mask_nonocc, s.d_max) for s in sets]
            points = ev.length_sweep(scenes, n_values, cfg, a.threshold)
            print("%6s  %9s  %12s" % ("n", "avg_error", "wall_seconds"))
            for p in points:
                print("%6d  %9.4f  %12.2f" % (p.n, p.avg_error, p.wall_time))
            if len(points) >= 2:
                print("linear fit of time vs n: R^2 = %.4f" % ev.linear_fit_r2([p.n for p in points],
                                                                             [p.wall_time for p in points]))
            ev.write_sweep_csv(a.out, points)
            bio.save_config(cfg, a.out + ".config.json")
        elif a.cmd == "radiometric":
            cfg.validate()
            rs = bio.load_radiometric_set(a.set, cfg.d_max, cfg.gt_scale)
            pattern = generate_pattern(cfg=cfg)
            m = ev.radiometric_protocol(rs.lefts, rs.rights, rs.gt, rs.mask_nonocc, pattern, cfg, a.threshold)
            print("%12s %8s %8s %8s" % ("left\\right", "c0", "c1", "c2"))
            for i in range(3):
                print("%12s %8.2f %8.2f %8.2f" % (f"c{i}", m.rate[i][0], m.rate[i][1], m.rate[i][2]))
            print("diagonal mean %.2f, off-diagonal mean %.2f" % (m.diagonal_mean(), m.off_diagonal_mean()))
            ev.write_radiometric_csv(a.out, m)
            bio.save_config(cfg, a.out + ".config.json")
        elif a.cmd == "bench":
            left, right = bio.load_image(a.left), bio.load_image(a.right)
            cfg.validate()
            pattern = generate_pattern(cfg=cfg)
            secs = ev.time_pipeline(left, right, pattern, cfg, a.runs)
            print("median of %d run%s: %.2f s (%dx%d, d_max=%d, n=%d, threads=%d)" % (
                a.runs, "" if a.runs == 1 else "s", secs, left.shape[1], left.shape[0], cfg.d_max, cfg.n,
                cfg.threads))
    except BsmError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
