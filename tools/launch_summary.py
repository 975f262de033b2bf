"""Summarise an ncu launch list (gpu__time_duration.sum per launch) into
per-kernel totals and shares.

    python tools/launch_summary.py launches.csv "<command>" > profiles/rNN_launches_<wl>.txt
"""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"^(void )?<unnamed>::", "", name)
    m = re.match(r"([A-Za-z0-9_]+)(<[^>]*>)?", name)
    return m.group(1) + (m.group(2) or "") if m else name[:40]


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
    launches = [(short(r[4]), float(r[14]) / 1e3) for r in rows if r[12] == "gpu__time_duration.sum"]
    cmd = sys.argv[2] if len(sys.argv) > 2 else "?"
    agg = collections.OrderedDict()
    for k, t in launches:
        agg.setdefault(k, []).append(t)
    tot = sum(t for _, t in launches)
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none: {cmd}")
    print("# (cold-cache, serialised launches: compare shares, not absolutes)")
    print(f"# {len(launches)} launches")
    print(f"{'kernel':32s} {'launches':>8s} {'total us':>11s} {'mean us':>10s} {'share':>7s}")
    for k, v in agg.items():
        print(f"{k:32s} {len(v):8d} {sum(v):11.1f} {sum(v) / len(v):10.1f} {100 * sum(v) / tot:6.1f}%")
    print(f"{'total':32s} {len(launches):8d} {tot:11.1f}")


if __name__ == "__main__":
    main()
