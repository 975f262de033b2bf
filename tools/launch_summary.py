"""Summarise an ncu launch list (gpu__time_duration.sum per launch) of
`tools/profile_pipeline.py <wl> 2` into per-kernel lines of the second pipeline.

    python tools/launch_summary.py launches.csv > profiles/rNN_launches_<wl>.txt
"""
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
    half = len(launches) // 2
    second = launches[half:]
    tot = sum(t for _, t in second)
    print("# ncu --metrics gpu__time_duration.sum --clock-control none, python tools/profile_pipeline.py c2 2")
    print("# (cold-cache, serialised launches: compare shares, not absolutes)")
    for k, t in second:
        print(f"{k:44s} {t:9.1f} us  {100 * t / tot:5.1f}%")
    print(f"{'total (second pipeline)':44s} {tot:9.1f} us")


if __name__ == "__main__":
    main()
