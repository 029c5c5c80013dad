"""Command-line front-ends over TNS1 files.

Mirrors the reference's `moba attend` and `moba bench` subcommands
(src/cli.py:108-161, :231-305) with the same flags, config-file merging
(JSON; unknown keys rejected; flags override the file, src/cli.py:54-68),
outputs and report JSON (src/report_schema.json), running the attention on
the GPU:

  python -m paper_2511_11571_b200.cli attend --q Q.tns --k K.tns --v V.tns --out O.tns \\
        [--block 128 --topk 8 --conv 3 --kernel W.tns --emit-plan plan.json --emit-lse lse.tns]
  python -m paper_2511_11571_b200.cli bench --n 2048,4096,8192 --block 128 --topk 8 --dim 64

`attend` output files carry the input dtype (the GPU computes in bf16 with
fp32 accumulation); `--emit-plan` writes counts / offsets / flat_queries
exactly as the reference (single-head inputs, src/cli.py:289-296). The
reference's `verify` and `snr` commands exercise its CPU oracle / SNR model
and are not part of the accelerated path.
"""

from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

from . import __version__
from .attention import moba_attention
from .core import ConfigError, MobaConfig, MobaError, OpCounters
from .keyconv import ConvKernel
from .tensorio import RunReport, Tensor, tensor_read, tensor_write, write_json_atomic


def _ints(text) -> list:
    return [int(x) for x in str(text).split(",") if x.strip()]


def _resolve(defaults: dict, config_path, args) -> dict:
    out = dict(defaults)
    if config_path:
        with open(config_path) as fh:
            cfg = json.load(fh)
        if not isinstance(cfg, dict):
            raise ConfigError("config file must hold a JSON object")
        unknown = set(cfg) - set(defaults)
        if unknown:
            raise ConfigError(f"unknown config keys {sorted(unknown)}")
        out.update(cfg)
    for key in defaults:
        val = getattr(args, key, None)
        if val is not None:
            out[key] = val
    return out


def _emit(report: RunReport) -> int:
    print(report.to_json())
    return 0 if report.passed else 1


def cmd_attend(args) -> int:
    defaults = {"q": None, "k": None, "v": None, "out": None, "block": 128, "topk": 8, "conv": 0, "kernel": None,
                "emit_plan": None, "emit_lse": None, "bq": 512, "br": None, "bc": None, "mode": "fp32"}
    r = _resolve(defaults, args.config, args)
    for name in ("q", "k", "v", "out"):
        if not r[name]:
            raise ConfigError(f"--{name} is required")
    Qt, Kt, Vt = tensor_read(r["q"]), tensor_read(r["k"]), tensor_read(r["v"])
    if not (Qt.dims == Kt.dims == Vt.dims):
        raise ConfigError(f"Q/K/V dims differ: {Qt.dims} {Kt.dims} {Vt.dims}")
    if Qt.array.ndim == 1:
        raise ConfigError("rank-1 tensors cannot carry (position, dim) data")
    conv = int(r["conv"])
    kernel = None
    if conv > 0:
        if not r["kernel"]:
            raise ConfigError("conv_width > 0 requires --kernel")
        kt = tensor_read(r["kernel"])
        if kt.array.ndim != 2 or kt.array.shape[0] != conv:
            raise ConfigError(f"kernel tensor must be {conv} x d, got {kt.dims}")
        kernel = ConvKernel(kt.array)
    if r["emit_plan"] and Qt.array.ndim == 3:
        raise ConfigError("--emit-plan is only supported for single-head (rank-2) inputs")
    Q, K, V = (t.array if t.array.ndim == 3 else t.array[None] for t in (Qt, Kt, Vt))
    N, d = Q.shape[1], Q.shape[2]
    cfg = MobaConfig(block_size_B=int(r["block"]), top_k=int(r["topk"]), head_dim_d=d,
                     logical_q_block_Bq=int(r["bq"]), phys_tile_Br=r["br"], phys_tile_Bc=r["bc"], conv_width=conv)
    counters = OpCounters()
    outs = np.empty_like(Q)
    lses = np.empty(Q.shape[:2], dtype=Q.dtype)
    plan = None
    t0 = time.perf_counter()
    for h in range(Q.shape[0]):
        # key conv fused with the centroids (routing on the unrounded K')
        res, plan = moba_attention(Q[h], K[h], V[h], cfg, counters, mode=r["mode"], kernel=kernel)
        outs[h] = res.output
        lses[h] = res.logsumexp
    elapsed = time.perf_counter() - t0
    tensor_write(Tensor(outs[0] if Qt.array.ndim == 2 else outs), r["out"])
    if r["emit_lse"]:
        tensor_write(Tensor(np.ascontiguousarray(lses[0] if Qt.array.ndim == 2 else lses)), r["emit_lse"])
    if r["emit_plan"]:
        write_json_atomic({"counts": np.asarray(plan.counts).reshape(-1).tolist(),
                           "offsets": np.asarray(plan.offsets).reshape(-1).tolist(),
                           "flat_queries": np.asarray(plan.flat_queries).reshape(-1).tolist()}, r["emit_plan"])
    report = RunReport("attend", {**r, "head_dim": d})
    report.metrics = {"n_tokens": float(N), "head_dim": float(d), "heads": float(Q.shape[0]),
                      "wall_seconds": elapsed, **{k: float(v) for k, v in counters.as_dict().items()}}
    report.passed = True
    return _emit(report)


def cmd_bench(args) -> int:
    """Counter sweep over sequence lengths (src/cli.py:108-161), timed on
    the GPU: routing + forward per N, the FLOP ratio against dense
    attention and the sparsity-band check for N >> kB."""
    defaults = {"n": "2048,4096,8192", "block": 128, "topk": 8, "dim": 64, "repeats": 3, "seed": 17}
    r = _resolve(defaults, args.config, args)
    n_list = _ints(r["n"])
    B, k, d = int(r["block"]), int(r["topk"]), int(r["dim"])
    for N in n_list:
        if N < B:
            raise ConfigError(f"N={N} is smaller than the block size {B}")
    cfg = MobaConfig(block_size_B=B, top_k=k, head_dim_d=d)
    rng = np.random.default_rng(int(r["seed"]))
    report = RunReport("bench", {**r, "n": n_list})
    m = {key: [] for key in ("attn_flops_moba", "attn_flops_dense", "flops_ratio", "score_flops", "gathered_elems",
                             "bulk_elems", "wall_seconds")}
    band_ok = True
    for N in n_list:
        Q, K, V = (rng.standard_normal((N, d)) for _ in range(3))
        counters = OpCounters()
        times = []
        for _ in range(int(r["repeats"])):
            counters.reset()
            t0 = time.perf_counter()
            moba_attention(Q, K, V, cfg, counters)
            times.append(time.perf_counter() - t0)
        dense = 2 * d * N * N                      # src/cli.py:103-105
        ratio = counters.attn_flops / dense
        for key, val in (("attn_flops_moba", counters.attn_flops), ("attn_flops_dense", dense),
                         ("flops_ratio", ratio), ("score_flops", counters.score_flops),
                         ("gathered_elems", counters.gathered_elems), ("bulk_elems", counters.bulk_elems),
                         ("wall_seconds", min(times))):
            m[key].append(float(val))
        if N >= 8 * k * B:
            band_ok = band_ok and abs(ratio * N / (k * B) - 1.0) <= 0.15
    report.metrics = {"n_values": [float(x) for x in n_list], **m}
    report.passed = band_ok
    return _emit(report)


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="paper_2511_11571_b200", description="B200 MoBA attention on TNS1 files")
    p.add_argument("--version", action="version", version=f"paper_2511_11571_b200 {__version__}")
    sub = p.add_subparsers(dest="command", required=True)
    a = sub.add_parser("attend", help="run routed attention on TNS1 tensor files (GPU)")
    for flag in ("q", "k", "v", "out", "kernel", "config"):
        a.add_argument(f"--{flag}")
    for flag in ("block", "topk", "bq", "br", "bc", "conv"):
        a.add_argument(f"--{flag}", type=int)
    a.add_argument("--emit-plan", dest="emit_plan")
    a.add_argument("--emit-lse", dest="emit_lse")
    a.add_argument("--mode", choices=["fp32", "tc"], help="routing score mode (fp32: parity, tc: tensor cores)")
    a.set_defaults(func=cmd_attend)
    b = sub.add_parser("bench", help="counter sweeps over sequence lengths (GPU)")
    b.add_argument("--n")
    for flag in ("block", "topk", "dim", "repeats", "seed"):
        b.add_argument(f"--{flag}", type=int)
    b.add_argument("--config")
    b.set_defaults(func=cmd_bench)
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except MobaError as exc:
        print(json.dumps({"error": type(exc).__name__, "message": str(exc)}), file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
