"""Instruction-level view of an ncu report around the hottest MUFU block:
each SASS line with its execution share and stall-sample share (the
softmax exp loop of the forward).
usage: python scripts/sass_region.py REPORT.ncu-rep [opcode=MUFU] [context=40]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
opc = sys.argv[2] if len(sys.argv) > 2 else "MUFU"
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
h = rows[hi]
si, ii, wi = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
stall_cols = [(j, c) for j, c in enumerate(h) if c.startswith("stall_") or "Stall" in c and c != h[wi]]
data = [r for r in rows[hi + 1:] if len(r) > ii]
tot = sum(float(r[ii] or 0) for r in data)
totw = sum(float(r[wi] or 0) for r in data) or 1
idx = [k for k, r in enumerate(data) if opc in r[si]]
best = max(idx, key=lambda k: float(data[k][ii] or 0))
lo, hi2 = max(0, best - ctx), min(len(data), best + ctx)
print(f"lines {lo}-{hi2} around the hottest {opc} (line {best}); columns: exec %, stall %")
for r in data[lo:hi2]:
    print(f"  {float(r[ii] or 0) / tot * 100:5.2f}% {float(r[wi] or 0) / totw * 100:5.2f}%  {r[si][:100]}")
