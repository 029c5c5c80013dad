"""Hot SASS lines of an ncu source export with per-reason stall samples.
usage: ncu -i X.ncu-rep --page source --csv --print-source sass > f.csv; python scripts/sass_hot.py f.csv [n]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; data = [r for r in rows[2:] if len(r) == len(h)]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
i_s = h.index("Warp Stall Sampling (All Samples)"); i_src = h.index("Source"); i_ex = h.index("Instructions Executed")
reasons = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
tot = sum(int(r[i_s] or 0) for r in data)
agg = {}
for r in data:
    for i in reasons:
        agg[h[i]] = agg.get(h[i], 0) + int(r[i] or 0)
print("total samples", tot, "by reason:", sorted(((v, k) for k, v in agg.items() if v), reverse=True)[:10])
for k, r in enumerate(sorted(data, key=lambda r: -int(r[i_s] or 0))[:n]):
    rs = sorted(((int(r[i] or 0), h[i][6:]) for i in reasons if int(r[i] or 0)), reverse=True)[:3]
    print(str(r[i_s]).rjust(6), str(r[i_ex]).rjust(8), r[0][-5:], r[i_src][:70].ljust(70), rs)
