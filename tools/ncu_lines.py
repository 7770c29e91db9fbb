"""Warp-stall samples and executed instructions per CUDA source line of one kernel:
ncu_lines.py report.ncu-rep kernel_regex[@n] [first_line last_line]
(@n picks the n-th matching kernel of the report, default 0)."""
import csv, io, subprocess, sys, collections
rep, kre = sys.argv[1], sys.argv[2]
nth = 0
if "@" in kre:
    kre, nth = kre.rsplit("@", 1)
    nth = int(nth)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if "Address" in r][nth]
h = rows[hi]
iss, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
agg = collections.defaultdict(lambda: [0, 0, ""])
for r in rows[hi + 1:]:
    if "Address" in r:
        break
    if len(r) != len(h) or not r[0].strip().isdigit():
        continue
    ln = int(r[0])
    agg[ln][0] += int(r[iss] or 0)
    agg[ln][1] += int(r[iex] or 0)
    agg[ln][2] = r[1]
tot = sum(v[0] for v in agg.values())
lo, hi2 = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 10**9)
print("samples", tot, "inst", sum(v[1] for v in agg.values()))
for ln in sorted(agg):
    s, x, src = agg[ln]
    if lo <= ln <= hi2 and (s > tot * 0.003 or x > 0):
        print(f"{ln:5d} {s:6d} {100*s/tot:5.1f}% {x:9d}  {src.strip()[:90]}")
