"""Attribute ncu warp-stall samples to CUDA source lines (innermost line in
the kernel's own .cu file, following 'inlined at' chains).

usage: python scripts/ncu_lines.py <report.ncu-rep> <cubin> <kernel.cu> [top] [mangled function name]
"""
import csv, io, re, subprocess, sys

rep, cubin, cu = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
fun = sys.argv[5] if len(sys.argv) > 5 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
ia, iall = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
base = min(int(r[ia], 16) for r in data)
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
cur, off2line = None, {}
in_fun = fun is None
for ln in dis.splitlines():
    if fun is not None and ln.lstrip().startswith(".text."):
        in_fun = fun in ln
        continue
    if not in_fun:
        continue
    if "//## File" in ln:
        # pick the first (file, line) pair on the line that is in our .cu
        pairs = re.findall(r'File "([^"]+)", line (\d+)', ln)
        mine = [int(l) for f, l in pairs if f.endswith(cu.split("/")[-1])]
        cur = mine[0] if mine else cur
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
agg = {}
for r in data:
    l = off2line.get(int(r[ia], 16) - base)
    agg[l] = agg.get(l, 0) + float(r[iall] or 0)
src = open(cu).read().split("\n")
tot = sum(agg.values())
for l, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{v:6.0f} {100 * v / tot:5.1f}%  L{l}: {src[l - 1].strip()[:90] if l else '?'}")
