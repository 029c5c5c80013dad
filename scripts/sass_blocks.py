"""Basic-block instruction accounting of an ncu report (SASS lines grouped by
equal execution count). usage: python scripts/sass_blocks.py REPORT [norm] [n]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
h = rows[hi]
si, ii = h.index("Source"), h.index("Instructions Executed")
wi = h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[hi + 1:] if len(r) > ii]
tot = sum(float(r[ii] or 0) for r in data)
totw = sum(float(r[wi] or 0) for r in data) or 1
print(f"total {tot:.3e} warp instructions")
blocks, cur = [], None
for k, r in enumerate(data):
    v = float(r[ii] or 0)
    if cur and cur[1] == v:
        cur[2] += 1
        cur[3].append(r[si].strip()[:44])
        cur[4] += float(r[wi] or 0)
    else:
        cur = [k, v, 1, [r[si].strip()[:44]], float(r[wi] or 0)]
        blocks.append(cur)
blocks.sort(key=lambda b: -b[1] * b[2])
for b in blocks[:nb]:
    print(f"line {b[0]:5d} n={b[2]:3d} exec/norm={b[1] / norm:8.2f} inst={b[1] * b[2] / tot * 100:5.1f}% stall={b[4] / totw * 100:5.1f}%  {b[3][0]} | {b[3][-1]}")
