"""Summarise an ncu --csv launch list (--metrics gpu__time_duration.sum[,dram__bytes_read.sum,
dram__bytes_write.sum]): per kernel, its share of the kernel time, launches, ms per launch and
DRAM GB read / written per launch.
python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

TIME_US = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6,
           "s": 1e6}
BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ii, ki, mi = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name")
    vi, ui = h.index("Metric Value"), h.index("Metric Unit")
    launches = collections.OrderedDict()  # id -> [name, us, rd, wr]
    for r in rows[hdr + 1:]:
        if len(r) <= max(ii, ki, mi, vi, ui):
            continue
        e = launches.setdefault(r[ii], [r[ki].split("(")[0][:70], 0.0, 0.0, 0.0])
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            e[1] += v * TIME_US[r[ui]]
        elif r[mi] == "dram__bytes_read.sum":
            e[2] += v * BYTES[r[ui]]
        elif r[mi] == "dram__bytes_write.sum":
            e[3] += v * BYTES[r[ui]]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for name, us, rd, wr in launches.values():
        a = agg[name]
        a[0] += 1
        a[1] += us
        a[2] += rd
        a[3] += wr
    tot = sum(v[1] for v in agg.values())
    print(f"# total kernel time {tot / 1e3:.1f} ms over {len(launches)} launches")
    print(" share launches   ms total  ms/launch  DRAM rd GB/launch  DRAM wr GB/launch  kernel")
    for n, (c, t, rd, wr) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{100 * t / tot:5.1f}% {c:8d} {t / 1e3:10.1f} {t / c / 1e3:10.3f} {rd / c / 1e9:18.3f} "
              f"{wr / c / 1e9:18.3f}  {n}")


if __name__ == "__main__":
    main(sys.argv[1])
