"""Top stall-sampled SASS lines of an ncu report (with --import-source).
usage: python scripts/ncu_top_stalls.py REPORT.ncu-rep [n]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
h = rows[hi]
si, ii, wi = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[hi + 1:] if len(r) > wi]
totw = sum(float(r[wi] or 0) for r in data) or 1

top = sorted(range(len(data)), key=lambda k: -float(data[k][wi] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]
for k in sorted(top):
    print(f"{k:5d} {float(data[k][wi] or 0)/totw*100:6.2f}%  {data[k][si][:90]}")
