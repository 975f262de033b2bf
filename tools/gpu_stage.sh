#!/bin/bash
# Per-stage device times on several workloads (tools/k3_ab.py prints wta only).
for wl in "$@"; do timeout 600 python tools/stage_ab.py $wl -1 2>&1 | tail -1; done
