"""profiles/traffic.json from the ncu DRAM-traffic CSVs of an evidence run
(tools/gpu_final3.sh / gpu_ncu_tail.sh): per workload, the bytes of one K3
launch (both directions) and of both views' mask launches.

    python tools/traffic_json.py <tag>     # reads gpurun_out/<tag>_traffic_<wl>.csv
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIZES = {"c1": (450, 375), "c2": (1392, 1104), "c3": (640, 480), "c4": (1920, 1080), "c5": (4096, 2160)}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    tag = sys.argv[1]
    out = {"k_cost_wta_tc": {}, "k_mask": {}, "_algorithmic_k_cost_wta_tc": {}}
    for wl, (w, h) in SIZES.items():
        tot = {}
        for r in csv.reader(open(os.path.join(ROOT, "gpurun_out", f"{tag}_traffic_{wl}.csv"))):
            if len(r) < 15 or r[0] == "ID" or r[12] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                continue
            k = "k_cost_wta_tc" if "k_cost_wta_tc" in r[4] else "k_mask"
            tot[k] = tot.get(k, 0.0) + float(r[14].replace(",", "")) * UNIT[r[13]]
        out["k_cost_wta_tc"][wl] = tot.get("k_cost_wta_tc")
        out["k_mask"][wl] = tot.get("k_mask")
        out["_algorithmic_k_cost_wta_tc"][wl] = 2 * w * h * 1536
    out["_source"] = (f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (gpurun_out/{tag}_traffic_<wl>.csv, "
                      "tools/traffic_json.py): k_cost_wta_tc = one launch (both directions); k_mask = the mask "
                      "launches of both views (reads are a few MB, the rest is the mask planes written, 512 B per "
                      "pixel per view, less where they stay in L2); _algorithmic_k_cost_wta_tc = 2 directions x W*H "
                      "x 1536 B (ref desc + ref mask + other desc, read once)")
    json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
