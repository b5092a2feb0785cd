"""Executed-instruction mix of one kernel from an ncu report's SASS source page:
python scripts/sass_mix.py report.ncu-rep [n_units]  (n_units: divide counts, e.g. pairs / 32)."""
import csv
import subprocess
import sys
from collections import Counter


def main(rep, units=None):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], text=True)
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ie = hdr.index("Instructions Executed")
    st = hdr.index("Warp Stall Sampling (All Samples)")
    cnt, stall = Counter(), Counter()
    for r in rows[2:]:
        if len(r) <= ie or not r[ie].strip():
            continue
        op = r[1].strip().split()
        if not op:
            continue
        name = op[0] if not op[0].startswith("@") else op[1]
        name = name.split(".")[0]
        cnt[name] += int(r[ie])
        stall[name] += int(r[st] or 0)
    tot = sum(cnt.values())
    ts = sum(stall.values())
    print(f"total warp instructions {tot:.4g}" + (f" = {tot / units:.1f} per unit" if units else ""))
    for k, v in cnt.most_common(30):
        print(f"  {k:10s} {v:14d} {100 * v / tot:5.1f}%" + (f"  {v / units:7.2f}/unit" if units else "")
              + f"  stall {100 * stall[k] / max(ts, 1):5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)
