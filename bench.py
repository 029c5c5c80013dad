#!/usr/bin/env python
"""Benchmark of the MoBA attention hot path (routing + fwd + bwd) on B200.

Contract (one JSON line on rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload = the metric's north-star point (BASELINE.json metric, paper Fig. 3
shape): batch 2 x 16 heads, N = 64K, d = 64, B = 128,
top-k 8, bf16 inputs resident in HBM (268 MB per tensor > the 126 MB L2;
L2 is also flushed between timed steps). A step = centroids + top-k routing
(tensor-core mode) + varlen plan + forward + backward (given dO), replayed as
one CUDA graph (MobaGraphedStep). Metric: TFLOP/s with the reference's
algorithmic FLOPs 14*d*P per head (P = visible (query, key) pairs,
tests/oracles.py:95-98) plus ms/step.

N > 1 (torchrun): the FIXED 32-head set is sharded over the ranks by
dist.shard_range (strong scaling, no collective in the timed region);
after timing, O / LSE / dQ / dK / dV are all-gathered over NCCL and rank 0
compares them with its own single-GPU run of all 32 heads.

At N = 1 rank 0 adds `sweep`: N = 8K ... 512K at the same b2 x h16 shape,
each point with MoBA ms / TFLOP/s, the dominant kernel's roofline and
FlashAttention-2 dense fwd+bwd at the same shape.

--impl reference: the unmodified reference package (baseline/_ref, its own
public API moba_attention + moba_backward, src/attention.py:305, :239) on
the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BATCH, HEADS, SEQ, DIM, BLOCK, TOPK = 2, 16, 65536, 64, 128, 8
SWEEP_N = (8192, 16384, 32768, 65536, 131072, 262144, 524288)
REF_PREFIX = 16384      # reference-arm sample: the causal 16K-token prefix of a 64K head
METRIC = "MoBA fwd+bwd ms and TFLOP/s vs seq len (B=128,k=8,d=64) vs FA2 dense & CPU ref"


def visible_pairs(N, B, k):
    # P = sum_i [min(k, i//B)*B + i%B + 1]  (tests/oracles.py:95-98)
    tot = 0
    for b in range(-(-N // B)):
        L = min(B, N - b * B)
        tot += L * min(k, b) * B + L * (L + 1) // 2
    return tot


def scored_candidates(N, B):
    return sum(min(B, N - b * B) * b for b in range(-(-N // B)))


def plan_entries(N, B, k):
    return sum(min(B, N - b * B) * (1 + min(k, b)) for b in range(-(-N // B)))


def step_flops(H, N, d, B, k):
    return 14 * d * visible_pairs(N, B, k) * H


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return j["hbm_gbs"], j["bf16_tflops"], "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.samples = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(device_index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0, t1):
        rows = [s for s in self.samples if t0 <= s[0] <= t1]
        window = "timed"
        if not rows:
            rows = [s for s in self.samples if s[0] >= t0 - 2.0]
            window = "timed+adjacent (timed region shorter than the 100 ms sampling period)"
        clocks, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for _, line in rows:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                clocks.append(float(parts[1]))
                maxes.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not clocks:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "window": "none"}
        clocks.sort()
        return {"sm_mhz": clocks[len(clocks) // 2], "sm_max_mhz": max(maxes), "reasons": sorted(reasons),
                "samples": len(clocks), "window": window}


# ----------------------------------------------------------------- reference (CPU) legs
def _ref_module():
    """The unmodified reference package shipped in baseline/_ref (pip
    --target install of /root/reference/pkg); None if absent."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "moba")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    import moba
    return moba


def _ref_head(args):
    """One head through the reference's public API: moba_attention (routing +
    forward, src/attention.py:305-314) then moba_backward (src/attention.py:
    239-302), f32 inputs, single-threaded. Returns wall seconds."""
    seed, N, d, B, k = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["MOBA_THREADS"] = "1"
    import numpy as np
    moba = _ref_module()
    rng = np.random.default_rng(seed)
    Q, K, V, dO = (rng.standard_normal((N, d)).astype(np.float32) for _ in range(4))
    cfg = moba.MobaConfig(block_size_B=B, top_k=k, head_dim_d=d)
    t = time.perf_counter()
    out, plan = moba.moba_attention(Q, K, V, cfg)
    moba.moba_backward(Q, K, V, out.output, dO, out.logsumexp, plan, cfg)
    return time.perf_counter() - t


def _oracle_head(args):
    seed, N, d, B, k = args
    import numpy as np
    from oracle import moba_oracle as orc
    rng = np.random.default_rng(seed)
    Q, K, V, dO = (rng.standard_normal((N, d)) for _ in range(4))
    t = time.perf_counter()
    plan = orc.build_plan(Q, K, B, k)
    O, L = orc.forward(Q, K, V, plan, B)
    orc.backward(Q, K, V, O, dO, L, plan, B)
    return time.perf_counter() - t


def _pool_run(fn, jobs, procs):
    import multiprocessing as mp
    for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS", "MOBA_THREADS"):
        os.environ[v] = "1"
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        pool.map(fn, [(1000 + i, 512, DIM, BLOCK, TOPK) for i in range(procs)])   # warm imports
        t0 = time.perf_counter()
        pool.map(fn, jobs)
        return time.perf_counter() - t0


def run_reference(args, rank, world):
    if rank != 0:
        return
    moba = _ref_module()
    fn, kind = (_ref_head, "reference") if moba is not None else (_oracle_head, "port")
    H = BATCH * HEADS
    procs = max(1, min(os.cpu_count() or 1, H))
    N = REF_PREFIX
    jobs = [(s, N, DIM, BLOCK, TOPK) for s in range(procs)]
    import multiprocessing as mp
    for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS", "MOBA_THREADS"):
        os.environ[v] = "1"
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        pool.map(fn, [(7 + i, 512, DIM, BLOCK, TOPK) for i in range(procs)])
        for _ in range(max(0, args.warmup)):
            pool.map(fn, jobs)
        tot = 0.0
        for _ in range(args.steps):
            t0 = time.perf_counter()
            pool.map(fn, jobs)
            tot += time.perf_counter() - t0
    flops = step_flops(procs, N, DIM, BLOCK, TOPK) * args.steps
    value = flops / tot / 1e12
    sample = (f"per step: {procs} heads (one per process) of the workload's causal {N}-token prefix "
              f"(queries 0..{N - 1} attend only keys < {N}, an exact sub-problem of each 64K head), "
              f"d={DIM} B={BLOCK} k={TOPK}, f32, through the reference's moba_attention + moba_backward "
              f"({'baseline/_ref' if kind == 'reference' else 'oracle port: baseline/_ref missing'}); "
              f"the reference's select_topk grows as N^2/B, so its prefix rate overstates its full-64K rate")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"b{BATCH} x h{HEADS}, N={SEQ}, d={DIM}, B={BLOCK}, top-k {TOPK}: routing + fwd + bwd "
                               f"(timed on a bounded sample, see cpu_baseline.sample)",
                   "parallelism": f"cpu x{procs} processes", "cpu_model": cpu_model()},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": procs, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_single_head():
    """One full 64K head of the workload through the reference on one core
    (~20 s): the reference's true per-head rate at the headline point."""
    moba = _ref_module()
    fn, kind = (_ref_head, "reference") if moba is not None else (_oracle_head, "port")
    wall = _pool_run(fn, [(0, SEQ, DIM, BLOCK, TOPK)], 1)
    return {"value": step_flops(1, SEQ, DIM, BLOCK, TOPK) / wall / 1e12, "unit": "TFLOP/s", "cores": 1,
            "kind": kind, "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
            "sample": f"one full head of the workload (N={SEQ}, d={DIM}, B={BLOCK}, k={TOPK}), f32, "
                      f"{'reference moba_attention + moba_backward (baseline/_ref)' if kind == 'reference' else 'f64 oracle port'}"
                      f", single core: {wall:.1f} s (the workload has {BATCH * HEADS} heads)"}


# ----------------------------------------------------------------- GPU arm helpers
def time_graph(gs, steps, flush, stream=None):
    import torch
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.zero_()                       # evict L2 between steps (untimed)
        evs[i][0].record()
        gs.replay()
        evs[i][1].record()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def stage_profile(mb, lib, _lib, q, k, v, do, B, topk, mode, flush, reps=2):
    """Per-stage device time of eager steps (CUDA-event stage timers on the
    launching stream inside libmoba_b200.so): {stage: (ms per launch, launches per step)}."""
    import torch
    qg, kg, vg = (t.clone().requires_grad_(True) for t in (q, k, v))
    torch.cuda.synchronize()
    lib.moba_timing_reset()
    lib.moba_timing_enable(1)
    for _ in range(reps):
        flush.zero_()
        for t in (qg, kg, vg):
            t.grad = None
        out = mb.moba_attn(qg, kg, vg, B, topk, mode=mode)
        out.backward(do)
    torch.cuda.synchronize()
    st = _lib.timing_read()
    lib.moba_timing_enable(0)
    return {s: (ms / max(n, 1), n / reps) for s, (ms, n) in st.items() if n > 0}


def roofline_of(stages, H, N, d, B, k, hbm, tc_peak, peak_src):
    """Dominant kernel's achieved rate vs its roofline. Algorithmic work per
    launch (one launch covers the rank's H heads):
    fwd 4dP, bwd 10dP, route 2dR FLOP; combine / centroid bytes."""
    P, R, E = visible_pairs(N, B, k), scored_candidates(N, B), plan_entries(N, B, k)
    n = -(-N // B)
    algo = {
        "fwd": ("tensor", 4 * d * P * H / 1e12, "TFLOP/s"),
        "bwd": ("tensor", 10 * d * P * H / 1e12, "TFLOP/s"),
        "route": ("tensor", 2 * d * R * H / 1e12, "TFLOP/s"),
        "combine": ("hbm", H * (E * (2 * d + 4) + N * (k + 1) * 4 + N * (2 * d + 4)) / 1e9, "GB/s"),
        "centroid": ("hbm", H * (2 * N * d + 4 * n * d) / 1e9, "GB/s"),
    }
    dom = max((s for s in stages if s in algo), key=lambda s: stages[s][0] * stages[s][1])
    bound, work, unit = algo[dom]
    avg_ms = stages[dom][0]
    achieved = work / (avg_ms / 1e3)
    peak = tc_peak if bound == "tensor" else hbm
    return {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
            "kernel": dom, "avg_ms": avg_ms,
            "peak_source": f"{peak_src} ({'bf16 dense burst' if bound == 'tensor' else 'HBM copy'})",
            "stage_ms_per_step": {s: round(v[0] * v[1], 4) for s, v in stages.items()}}


# ----------------------------------------------------------------- GPU arm
def run_ours(args, rank, world):
    import torch
    import torch.distributed as dist

    import paper_2511_11571_b200 as mb
    from paper_2511_11571_b200 import _lib
    from paper_2511_11571_b200.dist import gather_and_compare, shard_range

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    lib = _lib.load()
    Hg, N, d, B, k = BATCH * HEADS, SEQ, DIM, BLOCK, TOPK
    lo, hi = shard_range(Hg, world, rank)
    H = hi - lo
    gen = torch.Generator(device=dev).manual_seed(1234)        # the same global inputs on every rank
    full = [torch.randn(Hg, N, d, generator=gen, device=dev).bfloat16() for _ in range(4)]
    q, kk, v, do = (t[lo:hi].contiguous() for t in full)
    if world == 1:
        del full
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)

    # ---- the step captured once as a CUDA graph (MobaGraphedStep, the public
    # API for fixed-shape training loops) and replayed
    gs = mb.MobaGraphedStep((H, N, d), B, k, mode=args.route_mode, deterministic=args.deterministic)
    gs.step(q, kk, v, do)
    for _ in range(args.warmup):
        gs.replay()
    torch.cuda.synchronize()
    sampler = ClockSampler(dev.index) if rank == 0 else None
    time.sleep(0.3 if sampler else 0)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.time()
    ms_list = time_graph(gs, args.steps, flush)
    t1 = time.time()
    if world > 1:
        dist.barrier()
    ms = torch.tensor([sum(ms_list)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_max = float(ms.item())
    clocks = None
    if sampler:
        time.sleep(0.25)
        sampler.stop()
        clocks = sampler.summary(t0, t1)
    launches = gs.launches_per_step * args.steps
    flops_job = step_flops(Hg, N, d, B, k)
    value = flops_job * args.steps / (ms_max / 1e3) / 1e12

    # ---- multi-GPU verification (after timing): gather every rank's shard
    # over NCCL and compare with rank 0's single-GPU run of all heads
    verify = None
    if world > 1:
        local = {"O": gs.out.detach(), "LSE": gs.lse.detach(), "dQ": gs.q.grad, "dK": gs.k.grad, "dV": gs.v.grad}
        ref = None
        if rank == 0:
            xs = [t.clone().requires_grad_(True) for t in full[:3]]
            o, l = mb.moba_attn(*xs, B, k, mode=args.route_mode, deterministic=args.deterministic, return_lse=True)
            o.backward(full[3])
            ref = {"O": o.detach(), "LSE": l.detach(), "dQ": xs[0].grad, "dK": xs[1].grad, "dV": xs[2].grad}
        res = gather_and_compare(local, ref, Hg, dev)
        if rank == 0:
            verify = {nm: {"bitwise": b, "max_abs": m} for nm, (b, m) in res.items()}
            verify["note"] = ("O, LSE, dK, dV are deterministic kernels (bitwise); dQ under the parallel "
                              "schedule uses fp32 reduction atomics (order-dependent rounding)"
                              if not args.deterministic else "deterministic schedule: all bitwise")
        del full
    # ---- fp32-mode routing (the bit-exact parity router) timed beside the headline
    fp32_route = None
    if rank == 0 and args.route_mode == "tc" and not args.no_extra:
        g32 = mb.MobaGraphedStep((H, N, d), B, k, mode="fp32", deterministic=args.deterministic)
        g32.step(q, kk, v, do)
        g32.replay()
        t32 = time_graph(g32, max(3, min(args.steps, 10)), flush)
        fp32_route = {"ms_per_step": sum(t32) / len(t32),
                      "value": step_flops(H, N, d, B, k) / (sum(t32) / len(t32) / 1e3) / 1e12}
        del g32

    # ---- end to end through the public host-buffer API: pinned host Q, K,
    # V, dO in, host O, LSE, dQ, dK, dV out (copies inside the timed region)
    pin = [t.cpu().pin_memory() for t in (q, kk, v, do)]
    outs_h = (torch.empty((H, N, d), dtype=torch.bfloat16).pin_memory(),
              torch.empty((H, N), dtype=torch.float32).pin_memory(),
              *(torch.empty((H, N, d), dtype=torch.bfloat16).pin_memory() for _ in range(3)))
    e2e_ms = 0.0
    for i in range(args.warmup + args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        mb.moba_fwd_bwd_host(*pin, B, k, n_chunks=args.e2e_chunks, mode=args.route_mode,
                             deterministic=args.deterministic, out=outs_h, synchronize=False)
        b.record()
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_ms += a.elapsed_time(b)
    te = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_val = flops_job * args.steps / (float(te.item()) / 1e3) / 1e12
    h2d_bytes = sum(t.numel() * t.element_size() for t in pin)
    d2h_bytes = sum(t.numel() * t.element_size() for t in outs_h)
    del pin, outs_h

    # ---- roofline of the dominant kernel: per-stage device time measured on
    # the launching stream (library stage timers) in eager steps right after
    hbm, tc_peak, peak_src = load_peaks()
    stages = stage_profile(mb, lib, _lib, q, kk, v, do, B, k, args.route_mode, flush)
    roofline = roofline_of(stages, H, N, d, B, k, hbm, tc_peak, peak_src)
    roofline["traffic"] = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            if tj.get("workload") == f"b{BATCH}h{HEADS}_n{N}_d{d}" and world == 1:
                roofline["traffic"] = tj.get(roofline["kernel"])
                roofline["traffic_source"] = tj.get("source")
        except Exception:
            pass
    if rank != 0:
        return
    del gs, q, kk, v, do
    torch.cuda.empty_cache()

    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_baseline_single_head()
    sweep = None
    if world == 1 and not args.no_extra:
        sweep = run_sweep(args, dev, mb, lib, _lib, flush, hbm, tc_peak, peak_src,
                          headline={"N": N, "moba_ms": ms_max / args.steps, "roofline": roofline})

    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (torch.randn, seed 1234, the same global inputs on every rank)",
        "config": {"workload": f"metric north-star point: b{BATCH} x h{HEADS} = {Hg} heads, N={N}, d={d}, B={B}, "
                               f"top-k {k}; step = centroids + top-k routing ({args.route_mode}) + varlen + fwd + "
                               f"bwd, replayed as one CUDA graph (MobaGraphedStep)",
                   "batch": BATCH, "heads": HEADS, "seq_len": N, "head_dim": d, "block_size": B, "top_k": k,
                   "heads_per_gpu": H, "submission": "cuda_graph",
                   "parallelism": f"{Hg} heads sharded over {world} GPU(s) (dist.shard_range), no collective "
                                  f"in the timed region",
                   "bwd_schedule": "deterministic" if args.deterministic else "parallel",
                   "route_mode": args.route_mode,
                   "fp32_route_step": fp32_route,
                   "l2": "flushed (512 MB write) between timed steps; inputs 268 MB per tensor exceed L2",
                   "flops_per_step": flops_job, "launches_per_step": launches // max(args.steps, 1),
                   "multi_gpu_verify": verify},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d_bytes,
                "d2h_bytes_per_step": d2h_bytes, "ms_per_step": float(te.item()) / args.steps,
                "path": f"pinned host Q,K,V,dO -> moba_fwd_bwd_host (public API; {args.e2e_chunks or 'auto'} head chunks, "
                        f"H2D / one CUDA-graph replay per chunk / D2H on 3 streams) -> host O,LSE,dQ,dK,dV"},
        "gpu_launches": launches,
        "clocks": clocks,
        "sweep": sweep,
    }
    print(json.dumps(line), flush=True)


def time_cuda(fn, reps, flush):
    import torch
    tot = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        tot.append(a.elapsed_time(b))
    tot.sort()
    return tot[len(tot) // 2]


def run_sweep(args, dev, mb, lib, _lib, flush, hbm, tc_peak, peak_src, headline):
    """The metric's sequence-length sweep (paper Fig. 3: bsz 2, B=128, k=8;
    here 16 heads, d=64): per N the graphed MoBA step (median of reps), the
    dominant kernel's roofline, and FA2 dense fwd+bwd at the same shape."""
    import torch
    try:
        from flash_attn import flash_attn_func
    except Exception:  # pragma: no cover
        flash_attn_func = None
    Hg, d, B, k = BATCH * HEADS, DIM, BLOCK, TOPK
    points = []
    for N in SWEEP_N:
        if args.sweep_max and N > args.sweep_max:
            break
        gen = torch.Generator(device=dev).manual_seed(7)
        q, kk, v, do = (torch.randn(Hg, N, d, generator=gen, device=dev).bfloat16() for _ in range(4))
        rec = {"N": N}
        if N == headline["N"]:
            rec["moba_ms"] = headline["moba_ms"]
            roof = headline["roofline"]
        else:
            gs = mb.MobaGraphedStep((Hg, N, d), B, k, mode=args.route_mode)
            gs.step(q, kk, v, do)
            gs.replay()
            reps = 5 if N >= 131072 else 10
            t = sorted(time_graph(gs, reps, flush))
            rec["moba_ms"] = t[len(t) // 2]
            del gs
            torch.cuda.empty_cache()
            roof = roofline_of(stage_profile(mb, lib, _lib, q, kk, v, do, B, k, args.route_mode, flush, reps=1),
                               Hg, N, d, B, k, hbm, tc_peak, peak_src)
        rec["moba_tflops"] = step_flops(Hg, N, d, B, k) / (rec["moba_ms"] / 1e3) / 1e12
        rec["dominant"] = {x: roof[x] for x in ("kernel", "bound", "achieved", "unit", "frac", "avg_ms")}
        rec["stage_ms_per_step"] = roof["stage_ms_per_step"]
        if flash_attn_func is not None and not args.no_fa2:
            qf, kf, vf = (t.view(BATCH, HEADS, N, d).transpose(1, 2).contiguous().requires_grad_(True)
                          for t in (q, kk, v))
            dof = do.view(BATCH, HEADS, N, d).transpose(1, 2).contiguous()
            del q, kk, v, do
            torch.cuda.empty_cache()

            def fa2():
                for t in (qf, kf, vf):
                    t.grad = None
                o = flash_attn_func(qf, kf, vf, causal=True)
                o.backward(dof)

            fa2()
            fms = time_cuda(fa2, 2 if N >= 262144 else (3 if N >= 65536 else 10), flush)
            dense = 14 * d * N * (N + 1) // 2 * Hg
            rec.update({"fa2_dense_ms": fms, "fa2_dense_tflops": dense / (fms / 1e3) / 1e12,
                        "speedup_vs_fa2": fms / rec["moba_ms"]})
            del qf, kf, vf, dof
        points.append(rec)
        torch.cuda.empty_cache()
    return {"shape": f"b{BATCH} x h{HEADS}, d={d}, B={B}, top-k {k}, routing ({args.route_mode}) + fwd + bwd",
            "fa2": "flash_attn.flash_attn_func(causal=True) fwd+bwd, bf16 [b, N, h, d], median of reps, "
                   "FLOPs 14*d*N(N+1)/2 per head",
            "points": points}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--route-mode", choices=["fp32", "tc"], default="tc")
    ap.add_argument("--deterministic", action="store_true", help="deterministic dQ schedule")
    ap.add_argument("--e2e-chunks", type=int, default=None,
                    help="head chunks of the host-buffer pipeline (default: the API's own choice, ~32 MB of inputs each)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the sweep and the fp32-route step")
    ap.add_argument("--no-fa2", action="store_true")
    ap.add_argument("--sweep-max", type=int, default=0, help="largest N of the sweep (0 = 512K)")
    args = ap.parse_args()
    if args.impl == "ours":
        args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    try:
        run_ours(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
