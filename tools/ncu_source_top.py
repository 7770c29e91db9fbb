"""Top stalled SASS lines of one kernel in an ncu report: ncu_source_top.py rep kernel_regex [n [launch_skip]]"""
import csv, subprocess, sys, io
rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
skip = ["--launch-skip", sys.argv[4], "--launch-count", "1"] if len(sys.argv) > 4 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", *skip, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
h = rows[hi]
isrc, iss, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
body = [r for r in rows[hi + 1:] if len(r) == len(h) and r[iss].isdigit()]
tot = sum(int(r[iss] or 0) for r in body)
print("samples", tot)
top = sorted(range(len(body)), key=lambda i: -int(body[i][iss] or 0))[:n]
for i in sorted(top):
    r = body[i]
    print(f"{i:5d} {int(r[iss] or 0):7d} {int(r[iex] or 0):9d}  {r[isrc].strip()[:100]}")
