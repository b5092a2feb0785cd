"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import csv
import sys


def main(path, out, title):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    agg = {}
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        ms = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        agg.setdefault(name, [0, 0.0])
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(v[1] for v in agg.values())
    with open(out, "w") as f:
        f.write(title + "\n(cold-cache, serialised launches: compare SHARES, not absolutes)\n")
        for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{k[:90]:90s} launches={n:5d} total_ms={ms:10.3f} mean_ms={ms / n:9.4f} share={100 * ms / tot:6.2f}%\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
