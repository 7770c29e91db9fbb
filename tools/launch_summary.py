"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        name = r[ki].split("(")[0][:70]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale[r[ui]]
    tot = sum(v[1] for v in agg.values())
    print(f"total {tot / 1e3:.3f} ms over {sum(v[0] for v in agg.values())} launches")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t / 1e3:9.3f} ms {100 * t / tot:5.1f}%  n={c:4d}  avg={t / c:10.1f} us  {n}")


if __name__ == "__main__":
    main(sys.argv[1])
