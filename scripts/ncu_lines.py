"""Per-source-line executed warp instructions and stall samples of one kernel
(ncu --page source --print-source cuda,sass); python scripts/ncu_lines.py rep [units] [top]."""
import csv
import subprocess
import sys


def main(rep, units=1.0, top=40):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"], text=True)
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ie = hdr.index("Instructions Executed")
    st = hdr.index("Warp Stall Sampling (All Samples)")
    items = []
    for r in rows[2:]:
        try:
            n = int(r[ie] or 0)
            sm = int(r[st] or 0)
        except (ValueError, IndexError):
            continue
        if n:
            items.append((n, sm, r[0], r[1].strip()[:110]))
    tot = sum(i[0] for i in items)
    tots = sum(i[1] for i in items) or 1
    for n, sm, line, src in sorted(items, reverse=True)[:top]:
        print(f"{n / units:8.2f} {100 * n / tot:5.1f}% stall {100 * sm / tots:5.1f}%  L{line}: {src}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0, int(sys.argv[3]) if len(sys.argv) > 3 else 40)
