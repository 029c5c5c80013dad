"""Per-item timeline of CTA 0 of the forward kernel (clock64, MOBA_FWD_TRACE)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200 import _device
H, N, d, B, k = (int(x) for x in os.environ.get("CFG", "16,8192,64,128,8").split(","))
torch.manual_seed(0)
q, kk, v = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(3))
cent, _ = _device.centroids(kk, B)
plan = _device.route(q, cent, B, k, mode=1)
for _ in range(2): _device.fwd(q, kk, v, plan, d ** -0.5)
torch.cuda.synchronize()
path = "/tmp/fwd_trace.bin"
os.environ["MOBA_FWD_TRACE"] = path
_device.fwd(q, kk, v, plan, d ** -0.5)
torch.cuda.synchronize()
t = np.fromfile(path, dtype=np.int64).reshape(256, 16)
if not t.any():
    sys.exit("empty timeline: the product build compiles the recording out; build a timeline "
             "library (scripts/README.md: make -C var_tl/csrc EXTRA=-DMOBA_TIMELINE) and point MOBA_LIB at it")
t0 = t[t > 0].min()
names = ["mma:q_wait0", "mma:q_ok", "mma:p_wait0", "mma:p_ok", "pr:qe_wait0", "pr:qe_ok", "pr:issued",
         "sm:s_wait0", "sm:s_ok", "sm:p_done", "sm:o_ok", "sm:epi_done", "mma:pv_iss", "mma:s_iss", "sm:o_ld", "pr:ids_iss"]
print("li  " + " ".join(f"{n:>11s}" for n in names))
rows = [i for i in range(256) if t[i].any()]
for i in rows[:int(os.environ.get("ROWS", 24))]:
    print(f"{i:3d} " + " ".join(f"{(t[i, e] - t0) if t[i, e] else -1:11d}" for e in range(16)))
n = len(rows)
span = t[rows].max() - t0
print(f"items {n}, span {span} cycles, {span / max(n, 1):.0f} cycles/item")
d = lambda a, b: np.median([t[i, b] - t[i, a] for i in rows if t[i, a] and t[i, b]])
print("median: softmax (s_ok->p_done)", d(8, 9), " o wait (p_done->o_ok)", d(9, 10), " epilogue", d(10, 11),
      " s wait", d(7, 8), " mma p wait", d(2, 3), " prod qe wait", d(4, 5), " prod issue", d(5, 6))
# producer warp 0 loop: issue span and the gap from its last cp.async to the
# next item's q_empty check (item records, id loads, K/V TMA issue)
loop = [t[i + 1, 4] - t[i, 4] for i in rows if i + 1 in rows and t[i, 4] and t[i + 1, 4]]
gap = [t[i + 1, 4] - t[i, 6] for i in rows if i + 1 in rows and t[i, 6] and t[i + 1, 4]]
if loop:
    pct = lambda a: " / ".join(f"{np.percentile(a, p):.0f}" for p in (10, 50, 90, 99))
    print("producer loop p10/50/90/99:", pct(loop), "  post-issue gap:", pct(gap), "  mean loop", f"{np.mean(loop):.0f}")
ids = [t[i, 15] - t[i, 6] for i in rows if t[i, 15] and t[i, 6]]
top = [t[i + 1, 4] - t[i, 15] for i in rows if i + 1 in rows and t[i, 15] and t[i + 1, 4]]
if ids:
    print("producer: issued -> ids issued", pct(ids), "  ids issued -> next q_empty check", pct(top))
