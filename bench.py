#!/usr/bin/env python
"""Benchmark of the MoBA attention hot path (routing + fwd + bwd) on B200.

Contract (one JSON line on rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Under torchrun (N > 1) every rank runs its own heads (batch x heads shard
over GPUs, no collective in the timed region; max-over-ranks timing).

Workload (BASELINE.json configs[1]): per GPU 16 heads, N=8192, d=64, B=128,
top-k 8, bf16 inputs resident in HBM; a "step" = centroids + top-k routing +
varlen plan + forward + backward (given dO) over those heads. L2 (126 MB) is
flushed between timed steps (the inputs are 16 MB each). Metric: MoBA
fwd+bwd TFLOP/s with the reference's algorithmic FLOPs 14*d*P per head
(P = visible (query, key) pairs, tests/oracles.py:95-98), plus ms/step.

--impl reference: the CPU oracle port (oracle/, the restatement of the
reference's algorithm) on the box's host cores, one head per process,
rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HEADS, SEQ, DIM, BLOCK, TOPK = 16, 8192, 64, 128, 8
METRIC = "MoBA fwd+bwd ms and TFLOP/s vs seq len (B=128,k=8,d=64) vs FA2 dense & CPU ref"


def visible_pairs(N, B, k):
    # tests/oracles.py:95-98
    full = N // B
    tot = 0
    for b in range(-(-N // B)):
        L = min(B, N - b * B)
        tot += L * min(k, b) * B + L * (L + 1) // 2
    return tot


def scored_candidates(N, B):
    return sum(min(B, N - b * B) * b for b in range(-(-N // B)))


def step_flops(H, N, d, B, k):
    return 14 * d * visible_pairs(N, B, k) * H


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return j["hbm_gbs"], j["bf16_tflops"], j.get("bf16_tflops_sustained"), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.samples = []
        self.marks = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(device_index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
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


# ----------------------------------------------------------------- reference arm (CPU oracle)
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


def cpu_oracle_run(n_heads, procs, N=SEQ, d=DIM, B=BLOCK, k=TOPK, seed0=0):
    """Wall time of n_heads oracle fwd+bwd heads over `procs` worker processes."""
    import multiprocessing as mp
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["MKL_NUM_THREADS"] = "1"
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        pool.map(_oracle_head, [(seed0 + 1000 + i, 512, d, B, k) for i in range(procs)])  # warm imports
        t0 = time.perf_counter()
        pool.map(_oracle_head, [(seed0 + i, N, d, B, k) for i in range(n_heads)])
        return time.perf_counter() - t0


def run_reference(args, rank, world):
    if rank != 0:
        return
    procs = max(1, min(os.cpu_count() or 1, HEADS))
    per_head = step_flops(1, SEQ, DIM, BLOCK, TOPK)
    for _ in range(max(0, args.warmup)):
        cpu_oracle_run(procs, procs, seed0=7)
    tot = 0.0
    for s in range(args.steps):
        tot += cpu_oracle_run(procs, procs, seed0=100 * s)
    flops = per_head * procs * args.steps
    value = flops / tot / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3 * HEADS / procs,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "configs[1]: 16 heads x N=8192, d=64, B=128, top-k 8, routing+fwd+bwd",
                   "parallelism": f"cpu x{procs} processes"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": procs, "kind": "port",
                         "sample": f"{procs} heads (one per process) of N={SEQ} d={DIM} B={BLOCK} k={TOPK}, "
                                   f"numpy f64 oracle (oracle/moba_oracle.py), OPENBLAS_NUM_THREADS=1, "
                                   f"per step; ms_per_step scaled to 16 heads"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm
def run_ours(args, rank, world):
    import torch
    import torch.distributed as dist

    import paper_2511_11571_b200 as mb
    from paper_2511_11571_b200 import _lib

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    lib = _lib.load()
    H, N, d, B, k = HEADS, SEQ, DIM, BLOCK, TOPK
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    q, kk, v, do = (torch.randn(H, N, d, generator=gen, device=dev).bfloat16() for _ in range(4))
    qg, kg, vg = (t.detach().clone().requires_grad_(True) for t in (q, kk, v))
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def step(qx, kx, vx, dox):
        for t in (qx, kx, vx):
            t.grad = None
        out = mb.moba_attn(qx, kx, vx, B, k, mode=args.route_mode, deterministic=args.deterministic)
        out.backward(dox)
        return out

    for _ in range(args.warmup):
        step(qg, kg, vg, do)
    torch.cuda.synchronize()

    sampler = ClockSampler(dev.index) if rank == 0 else None
    time.sleep(0.3 if sampler else 0)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    lib.moba_timing_reset()
    lib.moba_timing_enable(1)
    launches0 = lib.moba_launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_wall0 = time.time()
    for i in range(args.steps):
        flush.zero_()                       # evict L2 between steps (untimed)
        evs[i][0].record()
        step(qg, kg, vg, do)
        evs[i][1].record()
    torch.cuda.synchronize()
    t_wall1 = time.time()
    if world > 1:
        dist.barrier()
    launches = int(lib.moba_launch_count() - launches0)
    stages = _lib.timing_read()
    lib.moba_timing_enable(0)
    ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    clocks = None
    if sampler:
        time.sleep(0.25)
        sampler.stop()
        clocks = sampler.summary(t_wall0, t_wall1)

    flops_rank = step_flops(H, N, d, B, k)
    eager_ms = ms_max
    eager_value = flops_rank * world * args.steps / (eager_ms / 1e3) / 1e12

    # ---- the same step replayed as one CUDA graph (MobaGraphedStep: the
    # public API for fixed-shape training loops); this is the headline value
    graph_info = None
    if not args.no_graph:
        gs = mb.MobaGraphedStep((H, N, d), B, k, mode=args.route_mode, deterministic=args.deterministic)
        gs.step(q, kk, v, do)
        for _ in range(args.warmup):
            gs.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        gevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        sampler_g = ClockSampler(dev.index) if rank == 0 else None
        time.sleep(0.3 if sampler_g else 0)
        tg0 = time.time()
        for i in range(args.steps):
            flush.zero_()
            gevs[i][0].record()
            gs.replay()
            gevs[i][1].record()
        torch.cuda.synchronize()
        tg1 = time.time()
        gms = torch.tensor([sum(a.elapsed_time(b) for a, b in gevs)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(gms, op=dist.ReduceOp.MAX)
        if sampler_g:
            time.sleep(0.25)
            sampler_g.stop()
            clocks = sampler_g.summary(tg0, tg1)
        # parity of the replay against the eager step (same inputs)
        out_e = mb.moba_attn(q, kk, v, B, k, mode=args.route_mode)
        graph_info = {"ms_per_step": float(gms.item()) / args.steps,
                      "launches_per_step": gs.launches_per_step,
                      "max_abs_vs_eager_out": float((gs.out.float() - out_e.float()).abs().max().item())}
        ms_max = float(gms.item())
        launches = gs.launches_per_step * args.steps
        del gs
    value = flops_rank * world * args.steps / (ms_max / 1e3) / 1e12

    # ---- end to end through the public host-buffer API: pinned host Q, K, V, dO
    # in, host O, LSE, dQ, dK, dV out; heads pipelined over copy/compute streams
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
    e2e_val = flops_rank * world * args.steps / (float(te.item()) / 1e3) / 1e12
    h2d_bytes = sum(t.numel() * t.element_size() for t in pin)
    d2h_bytes = sum(t.numel() * t.element_size() for t in outs_h)

    if rank != 0:
        return

    # ---- roofline of the dominant kernel (stage timers, same timed region)
    hbm, tc_burst, tc_sus, peak_kind = load_peaks()
    P = visible_pairs(N, B, k)
    R = scored_candidates(N, B)
    E = sum(1 + min(k, i // B) for i in range(0, N))
    algo = {  # algorithmic work per launch (one launch covers all H heads)
        "fwd": ("tensor", 4 * d * P * H / 1e12, "TFLOP/s"),
        "bwd": ("tensor", 10 * d * P * H / 1e12, "TFLOP/s"),
        "route": ("tensor", 2 * d * R * H / 1e12, "TFLOP/s"),
        "combine": ("hbm", H * (E * (2 * d + 4) + N * (k + 1) * 4 + N * (2 * d + 4)) / 1e9, "GB/s"),
        "centroid": ("hbm", H * (2 * N * d + 4 * (-(-N // B)) * d) / 1e9, "GB/s"),
    }
    stage_ms = {s: (v_[0] / max(v_[1], 1), v_[1]) for s, v_ in stages.items() if v_[1] > 0}
    dom = max((s for s in stage_ms if s in algo), key=lambda s: stage_ms[s][0] * stage_ms[s][1])
    bound, work, unit = algo[dom]
    avg_ms = stage_ms[dom][0]
    achieved = work / (avg_ms / 1e3)
    peak = tc_burst if bound == "tensor" else hbm
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(dom)
        except Exception:
            traffic = None
    roofline = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
                "traffic": traffic, "kernel": dom, "avg_ms": avg_ms,
                "peak_source": f"MEASURED_PEAKS.json ({peak_kind}, burst)" if bound == "tensor"
                else f"MEASURED_PEAKS.json ({peak_kind})",
                "stage_ms_per_step": {s: round(v_[0] * v_[1] / args.steps, 4) for s, v_ in stage_ms.items()}}

    # ---- CPU baseline (oracle port) and FA2 dense comparator
    cpu = None
    if world == 1 and not args.no_cpu:
        procs = max(1, min(os.cpu_count() or 1, H))
        wall = cpu_oracle_run(procs, procs)
        cpu = {"value": step_flops(1, N, d, B, k) * procs / wall / 1e12, "unit": "TFLOP/s", "cores": procs,
               "kind": "port",
               "sample": f"{procs} heads (one per process) of configs[1] (N={N}, d={d}, B={B}, k={k}) "
                         f"routing+fwd+bwd in the f64 numpy oracle, {wall:.1f} s wall"}
    extra = {}
    if not args.no_extra:
        extra = extra_measurements(args, dev, mb, flush)

    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (torch.randn, seeded per rank)",
        "config": {"workload": f"configs[1]: {H} heads/GPU x N={N}, d={d}, B={B}, top-k {k}; step = centroids + "
                               f"top-k routing ({args.route_mode}) + varlen + fwd + bwd"
                               + (", replayed as one CUDA graph (MobaGraphedStep)" if graph_info else ", eager"),
                   "submission": "cuda_graph" if graph_info else "eager",
                   "eager": {"ms_per_step": eager_ms / args.steps, "value": eager_value},
                   "graph": graph_info,
                   "heads_per_gpu": H, "seq_len": N, "head_dim": d, "block_size": B, "top_k": k,
                   "parallelism": f"heads sharded over {world} GPU(s), no collective",
                   "bwd_schedule": "deterministic" if args.deterministic else "parallel",
                   "l2": "flushed (512 MB write) between timed steps",
                   "flops_per_step_per_gpu": flops_rank},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d_bytes,
                "d2h_bytes_per_step": d2h_bytes, "ms_per_step": float(te.item()) / args.steps,
                "path": f"pinned host Q,K,V,dO -> moba_fwd_bwd_host (public API; {args.e2e_chunks} head chunks, "
                        f"H2D / one CUDA-graph replay per chunk / D2H on 3 streams) -> host O,LSE,dQ,dK,dV"},
        "gpu_launches": launches,
        "clocks": clocks,
        "extra": extra,
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


def extra_measurements(args, dev, mb, flush):
    """FA2 dense at the headline shape and the north-star point (N=64K,
    b2 x h16, d=64, B=128, k=8) for MoBA and FA2."""
    import torch
    out = {}
    try:
        from flash_attn import flash_attn_func
    except Exception as e:  # pragma: no cover
        flash_attn_func = None
        out["fa2_error"] = str(e)[:200]
    for tag, H, N in (("n8k_h16", HEADS, SEQ), ("n64k_b2h16", 32, 65536)):
        gen = torch.Generator(device=dev).manual_seed(7)
        q, kk, v, do = (torch.randn(H, N, DIM, generator=gen, device=dev).bfloat16() for _ in range(4))
        qg, kg, vg = (t.clone().requires_grad_(True) for t in (q, kk, v))

        def moba():
            for t in (qg, kg, vg):
                t.grad = None
            o = mb.moba_attn(qg, kg, vg, BLOCK, TOPK, mode=args.route_mode)
            o.backward(do)

        moba()
        reps = 5 if N > 16384 else 10
        ms = time_cuda(moba, reps, flush)
        rec = {"moba_ms": ms, "moba_tflops": step_flops(H, N, DIM, BLOCK, TOPK) / (ms / 1e3) / 1e12}
        if flash_attn_func is not None:
            qf, kf, vf = (t.transpose(0, 1).unsqueeze(0).contiguous().requires_grad_(True) for t in (q, kk, v))
            dof = do.transpose(0, 1).unsqueeze(0).contiguous()

            def fa2():
                for t in (qf, kf, vf):
                    t.grad = None
                o = flash_attn_func(qf, kf, vf, causal=True)
                o.backward(dof)

            fa2()
            fms = time_cuda(fa2, 3 if N > 16384 else 10, flush)
            dense = 14 * DIM * N * (N + 1) // 2 * H
            rec.update({"fa2_dense_ms": fms, "fa2_dense_tflops": dense / (fms / 1e3) / 1e12,
                        "speedup_vs_fa2": fms / ms})
            del qf, kf, vf, dof
        out[tag] = rec
        del q, kk, v, do, qg, kg, vg
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--route-mode", choices=["fp32", "tc"], default="tc")
    ap.add_argument("--deterministic", action="store_true", help="deterministic dQ schedule")
    ap.add_argument("--e2e-chunks", type=int, default=8, help="head chunks of the host-buffer pipeline")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="headline from eager launches instead of a CUDA graph")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
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
