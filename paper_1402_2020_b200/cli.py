"""Command-line front end over the GPU pipeline.

``python -m paper_1402_2020_b200 ...`` runs the C++ tool
``paper_1402_2020_b200/bsm`` (csrc/bsm_cli.cpp over the include/bsm drop-in
headers), the single implementation of the reference tool's subcommands,
flags, output files and printed lines (tools/bsm.cpp:93-246):

    match LEFT RIGHT OUT [--stages] [--pattern P] [--emit-pattern P] ...
    eval RESULT GT [--nonocc M] [--all M] [--disc M] [--threshold T]
    sweep SCENE_DIR... [--n_values 512,1024] [--out CSV]
    radiometric SET_DIR [--out CSV]
    bench LEFT RIGHT [--runs K]

plus the shared config flags (--config, --n, --S, --spread, --seed, --d_max,
--lambda_c, --lambda_e, --lr_tolerance, --vote_radius, --gt_scale, --threads).
"""
from __future__ import annotations

import os
import subprocess
import sys
from typing import List, Optional

TOOL = os.path.join(os.path.dirname(os.path.abspath(__file__)), "bsm")


def main(argv: Optional[List[str]] = None) -> int:
    args = sys.argv[1:] if argv is None else list(argv)
    if not os.path.exists(TOOL):
        print(f"error: {TOOL} is missing: run __graft_entry__.build()", file=sys.stderr)
        return 2
    sys.stdout.flush()
    return subprocess.call([TOOL, *args])
