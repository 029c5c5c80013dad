"""Aggregate an ncu gpu__time_duration launch list (CSV): per-kernel total over
the second half of the launches (the last of two identical steps)."""
import csv, io, sys
txt = open(sys.argv[1]).read()
txt = txt[txt.index('"ID"'):]
rows = [r for r in csv.DictReader(io.StringIO(txt)) if r["Metric Name"] == "gpu__time_duration.sum"]
half = rows[len(rows) // 2:]
agg = {}
for r in half:
    k = r["Kernel Name"].split("(")[0][-60:]
    agg[k] = agg.get(k, 0.0) + float(r["Metric Value"].replace(",", ""))
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{v / 1e3:10.1f} us  {100 * v / tot:5.1f}%  {k}")
print(f"{tot / 1e3:10.1f} us  total")
