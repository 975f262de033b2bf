"""Print a compact text summary of an ncu report (key throughput metrics,
pipe utilisation, stall reasons, DRAM traffic per launch).

    python tools/summarize_ncu.py report.ncu-rep [kernel-regex]
"""
import csv
import subprocess
import sys

WANT = ["Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Theoretical Active Warps per SM",
        "Achieved Active Warps Per SM", "Eligible Warps Per Scheduler", "Block Size", "Grid Size",
        "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else None
    kargs = ["-k", "regex:" + kre] if kre else []
    rows = list(csv.reader(run([rep, "--page", "details", "--csv"] + kargs).splitlines()))
    hdr = rows[0]
    ii, ki, mi, vi, ui = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    seen, names = {}, {}
    for r in rows[1:]:  # keyed by launch ID: one report may hold several launches
        names[r[ii]] = r[ki]
        if r[mi] in WANT and (r[ii], r[mi]) not in seen:
            seen[(r[ii], r[mi])] = f"{r[vi]} {r[ui]}".strip()
    raw = list(csv.reader(run([rep, "--page", "raw", "--csv"] + kargs).splitlines()))
    h, units, vals = raw[0], raw[1], raw[2:]
    by_id = {v[h.index("ID")]: v for v in vals}
    for lid in sorted(names, key=int):
        k = names[lid]
        print(f"== {k[:110]}")
        for m in WANT:
            if (lid, m) in seen:
                print(f"   {m:36s} {seen[(lid, m)]}")
        if lid in by_id:
            v = by_id[lid]
            get = lambda name: float(v[h.index(name)].replace(",", "")) if name in h and v[h.index(name)] else None
            rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
            if rd is not None and wr is not None:
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                ur = scale.get(units[h.index("dram__bytes_read.sum")], 1)
                uw = scale.get(units[h.index("dram__bytes_write.sum")], 1)
                print(f"   {'dram bytes read + write':36s} {(rd * ur + wr * uw) / 1e6:.1f} MB per launch")
            pipes = []
            for i, name in enumerate(h):
                if name.startswith("sm__inst_executed_pipe_") and name.endswith("avg.pct_of_peak_sustained_active"):
                    x = get(name)
                    if x and x > 2:
                        pipes.append((x, name[len("sm__inst_executed_pipe_"):].split(".")[0]))
            if pipes:
                print("   pipes (% of peak, active):        " + ", ".join(f"{p} {x:.0f}" for x, p in sorted(pipes, reverse=True)))
            st = []
            for i, name in enumerate(h):
                if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
                    x = get(name)
                    if x:
                        st.append((x, name[len("smsp__pcsamp_warps_issue_stalled_"):]))
            tot = sum(x for x, _ in st) or 1
            print("   stalls (% of samples):            " +
                  ", ".join(f"{n2} {x / tot * 100:.0f}" for x, n2 in sorted(st, reverse=True)[:7]))


if __name__ == "__main__":
    main()
