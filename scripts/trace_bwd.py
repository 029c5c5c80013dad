"""Per-tile timeline of CTA 0 of the pipelined backward kernel (clock64, MOBA_BWD_TRACE)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11571_b200 import _device
H, N, d, B, k = (int(x) for x in os.environ.get("CFG", "16,8192,64,128,8").split(","))
torch.manual_seed(0)
q, kk, v, do = (torch.randn(H, N, d, device="cuda").bfloat16() for _ in range(4))
cent, _ = _device.centroids(kk, B)
plan = _device.route(q, cent, B, k, mode=1)
o, lse = _device.fwd(q, kk, v, plan, d ** -0.5)
for _ in range(2): _device.bwd(q, kk, v, o, do, lse, plan, d ** -0.5, deterministic=False)
torch.cuda.synchronize()
path = "/tmp/bwd_trace.bin"
os.environ["MOBA_BWD_TRACE"] = path
_device.bwd(q, kk, v, o, do, lse, plan, d ** -0.5, deterministic=False)
torch.cuda.synchronize()
t = np.fromfile(path, dtype=np.int64).reshape(256, 16)
if not t.any():
    sys.exit("empty timeline: the product build compiles the recording out; build a timeline "
             "library (scripts/README.md: make -C var_tl/csrc EXTRA=-DMOBA_TIMELINE) and point MOBA_LIB at it")
t0 = t[t > 0].min()
names = ["P:qe_wait0", "P:qe_ok", "P:issued", "M:s_issue", "M:p_ok", "M:mma_done", "S:s_wait0", "S:s_ok",
         "S:A_done", "S:dp_ok", "S:B_done", "E:dq_ok", "E:done", "M:dvdk", "M:dq"]
print("g   " + " ".join(f"{n:>10s}" for n in names))
rows = [i for i in range(256) if t[i].any()]
for i in rows[:int(os.environ.get("ROWS", 16))]:
    print(f"{i:3d} " + " ".join(f"{(t[i, e] - t0) if t[i, e] else -1:10d}" for e in range(15)))
n = len(rows)
span = t[rows].max() - t0
print(f"tiles {n}, span {span} cycles, {span / max(n, 1):.0f} cycles/tile")
d_ = lambda a, b: np.median([t[i, b] - t[i, a] for i in rows if t[i, a] and t[i, b]])
print("median: phaseA", d_(7, 8), " dp wait", d_(8, 9), " phaseB", d_(9, 10), " s wait", d_(6, 7),
      " mma p->issued", d_(4, 5), " dVdK issue", d_(4, 13), " dQ issue", d_(13, 14), " s_issue->p_ok", d_(3, 4), " prod qe wait", d_(0, 1), " prod issue", d_(1, 2), " epi (dq_ok->issued)", d_(11, 12))
