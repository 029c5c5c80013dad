"""Stall samples / executed instructions per window of W SASS lines (which role of a
warp-specialised kernel waits on what). usage: python scripts/ncu_stall_buckets.py REPORT.ncu-rep W"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]; W = int(sys.argv[2])
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
h = rows[hi]
si, ii, wi = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
sc = [(j, c) for j, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
data = [r for r in rows[hi + 1:] if len(r) > wi]
totw = sum(float(r[wi] or 0) for r in data) or 1
tot = sum(float(r[ii] or 0) for r in data) or 1
for b in range(0, len(data), W):
    seg = data[b:b + W]
    w = sum(float(r[wi] or 0) for r in seg)
    e = sum(float(r[ii] or 0) for r in seg)
    reasons = collections.Counter()
    for r in seg:
        for j, c in sc: reasons[c[6:]] += float(r[j] or 0)
    ops = collections.Counter(r[si].split()[1 if r[si].startswith('@') else 0].split('.')[0] for r in seg if r[si].split())
    if w / totw > 0.01:
        print(f"{b:5d}-{b+W-1:5d} stall {w/totw*100:5.1f}% exec {e/tot*100:5.1f}%  " + " ".join(f"{c}:{v/totw*100:.1f}" for c, v in reasons.most_common(3)) + "  ops " + ",".join(o for o, _ in ops.most_common(5)))
