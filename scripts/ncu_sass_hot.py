"""Per-instruction SASS hot list of an ncu report (source page): stall samples and executions."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], text=True,
                              stderr=subprocess.DEVNULL)
rows = list(csv.reader(raw.splitlines()))
hdr = rows[1]
data = rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
tot = sum(int(r[iS] or 0) for r in data)
mode = sys.argv[3] if len(sys.argv) > 3 else "list"
if mode == "list":
    for idx, r in enumerate(data):
        s = int(r[iS] or 0)
        print(f"{idx:5d} {s:7d} {100.0*s/tot:5.1f}% {int(r[iE] or 0):>12d}  {r[1].strip()}")
else:
    top = sorted(range(len(data)), key=lambda i: -int(data[i][iS] or 0))[:n]
    for idx in sorted(top):
        r = data[idx]
        s = int(r[iS] or 0)
        print(f"{idx:5d} {s:7d} {100.0*s/tot:5.1f}% {int(r[iE] or 0):>12d}  {r[1].strip()}")
