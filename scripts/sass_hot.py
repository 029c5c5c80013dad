"""SASS hot spots of an ncu report: opcode mix and the hottest instruction windows.
usage: python scripts/sass_hot.py REPORT.ncu-rep [window]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
W = int(sys.argv[2]) if len(sys.argv) > 2 else 24
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
h = rows[hi]
si, ii, wi = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[hi + 1:] if len(r) > ii]
tot = sum(float(r[ii] or 0) for r in data)
totw = sum(float(r[wi] or 0) for r in data) or 1
print(f"total warp instructions {tot:.3e}, {len(data)} SASS lines")
op, opw = collections.Counter(), collections.Counter()
for r in data:
    toks = r[si].split()
    if not toks:
        continue
    o = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    o = o.split(".")[0]
    op[o] += float(r[ii] or 0)
    opw[o] += float(r[wi] or 0)
print("opcodes:", ", ".join(f"{o} {c / tot * 100:.1f}%" for o, c in op.most_common(14)))
blk = collections.Counter()
for k, r in enumerate(data):
    blk[k // W] += float(r[ii] or 0)
for b, c in blk.most_common(6):
    print(f"--- window {b * W}-{b * W + W - 1}: {c / tot * 100:.1f}% of instructions")
    for r in data[b * W:b * W + W]:
        print(f"   {float(r[ii] or 0) / tot * 100:5.2f}% {float(r[wi] or 0) / totw * 100:5.2f}%st  {r[si][:90]}")
