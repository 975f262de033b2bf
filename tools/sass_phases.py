"""Dynamic instruction mix and per-phase shares of one kernel from an ncu report
(`--set full --import-source on`): the SASS page's per-instruction executed counts and
stall samples, split at the CTA barriers.  The opcode mix is exact; the segments are only a
guide: ptxas moves register-only work (e.g. the later bit planes' transposes in k_mask_q) across
barriers, so a segment is not a source-level phase.

    ncu -i rep.ncu-rep --page source --csv --kernel-name regex:k_mask_q > sass.csv
    python tools/sass_phases.py sass.csv > profiles/rNN_sass_<kernel>.txt
"""
import collections
import csv
import re
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    col = {n: i for i, n in enumerate(hdr)}
    ins, seen = [], set()
    for r in rows[hdr_i + 1:]:
        if len(r) < len(hdr) or not r[0].startswith("0x") or r[0] in seen:  # the page lists a kernel once per view
            continue
        seen.add(r[0])
        src = r[col["Source"]].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split()[0].rstrip(";")
        ins.append((op, int(r[col["Instructions Executed"]]), int(r[col["# Samples"]])))
    tot_i = sum(i for _, i, _ in ins)
    tot_s = sum(s for _, _, s in ins)
    print(f"# {rows[0][1][:90]}")
    print(f"# {len(ins)} SASS instructions, {tot_i:,} warp-instructions executed, {tot_s:,} stall samples\n")
    print("phase (between CTA barriers)   static  executed   share   samples share")
    ph, acc = 0, [0, 0, 0]
    for op, i, s in ins + [("BAR.SYNC.END", 0, 0)]:
        acc[0] += 1; acc[1] += i; acc[2] += s
        if op.startswith("BAR"):
            print(f"  segment {ph:2d} (ends at {op:<18}) {acc[0]:5d} {acc[1]:12,d} {100 * acc[1] / tot_i:6.1f}% {100 * acc[2] / max(tot_s, 1):6.1f}%")
            ph, acc = ph + 1, [0, 0, 0]
    print("\nopcode       executed   share   samples share")
    by = collections.defaultdict(lambda: [0, 0])
    for op, i, s in ins:
        k = ".".join(op.split(".")[:2]) if op.startswith(("IMAD", "LDS", "LDG", "STS", "STG")) else op.split(".")[0]
        by[k][0] += i; by[k][1] += s
    for k, (i, s) in sorted(by.items(), key=lambda kv: -kv[1][0])[:24]:
        print(f"  {k:<12} {i:12,d} {100 * i / tot_i:6.1f}% {100 * s / max(tot_s, 1):6.1f}%")


if __name__ == "__main__":
    main()
