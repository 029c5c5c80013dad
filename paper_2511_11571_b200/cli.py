"""Command-line front-ends over TNS1 files.

Two subcommands with the reference CLI's flags, config-file semantics and
report schema (src/cli.py, src/report_schema.json), executed on the GPU:

  python -m paper_2511_11571_b200.cli attend --q Q.tns --k K.tns --v V.tns --out O.tns \\
        [--block 128 --topk 8 --conv 3 --kernel W.tns --emit-plan plan.json --emit-lse lse.tns]
  python -m paper_2511_11571_b200.cli bench --n 2048,4096,8192 --block 128 --topk 8 --dim 64

Settings come in three layers: built-in defaults < a JSON object from
--config (keys must be known options) < flags given on the command line.
`attend` sends every head of a rank-3 [H, N, d] file through ONE batched
GPU call (routing, plan and attention for all heads at once) and writes the
outputs in the input's dtype; `--emit-plan` (rank-2 inputs only) writes the
plan's counts / offsets / flat_queries. `bench` sweeps sequence lengths and
reports the operation counters (closed forms, counters.py) and GPU wall
time. Every failure is a MobaError reported as JSON on stderr, exit code 2;
a report with passed=false exits 1.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import __version__
from .attention import moba_attention
from .core import ConfigError, MobaConfig, MobaError, OpCounters
from .keyconv import ConvKernel
from .tensorio import RunReport, Tensor, tensor_read, tensor_write, write_json_atomic


@dataclass(frozen=True)
class Option:
    """One setting: flag name (dashes in the flag, underscores in the
    settings dict), value type, default, whether a run needs it."""

    name: str
    kind: type = str
    default: object = None
    required: bool = False
    help: str = ""

    @property
    def flag(self) -> str:
        return "--" + self.name.replace("_", "-")


ATTEND = (
    Option("q", required=True, help="query tensor file (TNS1, [N, d] or [H, N, d])"),
    Option("k", required=True, help="key tensor file"),
    Option("v", required=True, help="value tensor file"),
    Option("out", required=True, help="output tensor file"),
    Option("block", int, 128, help="key block size B"),
    Option("topk", int, 8, help="routed past blocks per query (the own block is added)"),
    Option("conv", int, 0, help="key short-conv width (0, 3 or 5)"),
    Option("kernel", help="conv weight tensor file [conv, d]"),
    Option("emit_plan", help="write the routing plan as JSON (rank-2 inputs)"),
    Option("emit_lse", help="write the log-sum-exp tensor"),
    Option("bq", int, 512, help="logical query block (counter semantics only)"),
    Option("br", int, help="physical row tile (counter semantics only)"),
    Option("bc", int, help="physical column tile (counter semantics only)"),
    Option("mode", str, "fp32", help="routing scores: fp32 (parity) or tc (tensor cores)"),
)

BENCH = (
    Option("n", str, "2048,4096,8192", help="comma list of sequence lengths"),
    Option("block", int, 128),
    Option("topk", int, 8),
    Option("dim", int, 64),
    Option("repeats", int, 3),
    Option("seed", int, 17),
)


def settings(options, cli_args) -> dict:
    """defaults < --config JSON object < explicit flags."""
    values = {o.name: o.default for o in options}
    path = getattr(cli_args, "config", None)
    if path:
        with open(path) as fh:
            doc = json.load(fh)
        if not isinstance(doc, dict):
            raise ConfigError(f"{path}: expected a JSON object of settings")
        stray = sorted(set(doc) - set(values))
        if stray:
            raise ConfigError(f"{path}: unrecognised settings {stray}")
        values.update(doc)
    for o in options:
        given = getattr(cli_args, o.name, None)
        if given is not None:
            values[o.name] = given
    missing = [o.flag for o in options if o.required and not values[o.name]]
    if missing:
        raise ConfigError(f"missing required option(s): {', '.join(missing)}")
    return values


def _heads(t: Tensor) -> np.ndarray:
    return t.array if t.array.ndim == 3 else t.array[None]


def attend(s: dict) -> RunReport:
    q_t, k_t, v_t = tensor_read(s["q"]), tensor_read(s["k"]), tensor_read(s["v"])
    if len({q_t.dims, k_t.dims, v_t.dims}) != 1:
        raise ConfigError(f"Q, K and V must have equal dims, got {q_t.dims}, {k_t.dims}, {v_t.dims}")
    rank = q_t.array.ndim
    if rank == 1:
        raise ConfigError("attend needs (position, channel) data: rank-1 tensors are not accepted")
    if s["emit_plan"] and rank != 2:
        raise ConfigError("--emit-plan describes one head: pass rank-2 [N, d] inputs")
    width = int(s["conv"])
    kernel = None
    if width:
        if not s["kernel"]:
            raise ConfigError(f"a conv width of {width} needs the --kernel weight file")
        w = tensor_read(s["kernel"]).array
        if w.ndim != 2 or w.shape[0] != width:
            raise ConfigError(f"--kernel must hold a [{width}, d] tensor, got shape {w.shape}")
        kernel = ConvKernel(w)
    Q, K, V = _heads(q_t), _heads(k_t), _heads(v_t)
    H, N, d = Q.shape
    cfg = MobaConfig(block_size_B=int(s["block"]), top_k=int(s["topk"]), head_dim_d=d,
                     logical_q_block_Bq=int(s["bq"]), phys_tile_Br=s["br"], phys_tile_Bc=s["bc"],
                     conv_width=width)
    counters = OpCounters()
    t0 = time.perf_counter()
    # all heads in one batched call (torch views of the host arrays: the
    # reference-shaped numpy entry point takes one [N, d] head at a time)
    res, plan = moba_attention(*(torch.from_numpy(np.ascontiguousarray(x)) for x in (Q, K, V)), cfg, counters,
                               mode=s["mode"], kernel=kernel)
    out = res.output.float().cpu().numpy().astype(Q.dtype)
    lse = res.logsumexp.float().cpu().numpy().astype(Q.dtype)
    wall = time.perf_counter() - t0
    squeeze = (lambda a: a[0]) if rank == 2 else (lambda a: a)
    tensor_write(Tensor(np.ascontiguousarray(squeeze(out))), s["out"])
    if s["emit_lse"]:
        tensor_write(Tensor(np.ascontiguousarray(squeeze(lse))), s["emit_lse"])
    if s["emit_plan"]:
        write_json_atomic({name: np.asarray(getattr(plan, name)).reshape(-1).tolist()
                           for name in ("counts", "offsets", "flat_queries")}, s["emit_plan"])
    report = RunReport("attend", {**s, "head_dim": d})
    report.metrics = {"n_tokens": float(N), "head_dim": float(d), "heads": float(H), "wall_seconds": wall}
    report.metrics.update({name: float(val) for name, val in counters.as_dict().items()})
    report.passed = True
    return report


def bench(s: dict) -> RunReport:
    """Counter sweep over sequence lengths on the GPU. For N >= 8kB the
    routed/dense attention ratio must sit within 15% of kB/N (the
    reference's sparsity band check)."""
    lengths = [int(x) for x in str(s["n"]).split(",") if x.strip()]
    B, k, d = int(s["block"]), int(s["topk"]), int(s["dim"])
    short = [N for N in lengths if N < B]
    if short:
        raise ConfigError(f"sequence lengths {short} are shorter than the block size {B}")
    cfg = MobaConfig(block_size_B=B, top_k=k, head_dim_d=d)
    rng = np.random.default_rng(int(s["seed"]))
    cols = {c: [] for c in ("attn_flops_moba", "attn_flops_dense", "flops_ratio", "score_flops",
                            "gathered_elems", "bulk_elems", "wall_seconds")}
    in_band = True
    for N in lengths:
        Q, K, V = (rng.standard_normal((N, d)) for _ in range(3))
        best, counters = float("inf"), None
        for _ in range(max(1, int(s["repeats"]))):
            c = OpCounters()
            t0 = time.perf_counter()
            moba_attention(Q, K, V, cfg, c)
            best = min(best, time.perf_counter() - t0)
            counters = c
        dense = 2 * d * N * N
        ratio = counters.attn_flops / dense
        row = {"attn_flops_moba": counters.attn_flops, "attn_flops_dense": dense, "flops_ratio": ratio,
               "score_flops": counters.score_flops, "gathered_elems": counters.gathered_elems,
               "bulk_elems": counters.bulk_elems, "wall_seconds": best}
        for c_name, val in row.items():
            cols[c_name].append(float(val))
        if N >= 8 * k * B:
            in_band &= abs(ratio * N / (k * B) - 1.0) <= 0.15
    report = RunReport("bench", {**s, "n": lengths})
    report.metrics = {"n_values": [float(N) for N in lengths], **cols}
    report.passed = bool(in_band)
    return report


COMMANDS = {"attend": (ATTEND, attend, "routed attention on TNS1 tensor files (GPU)"),
            "bench": (BENCH, bench, "counter sweep over sequence lengths (GPU)")}


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2511_11571_b200", description="B200 MoBA attention on TNS1 files")
    parser.add_argument("--version", action="version", version=f"paper_2511_11571_b200 {__version__}")
    sub = parser.add_subparsers(dest="command", required=True)
    for name, (options, _, text) in COMMANDS.items():
        sp = sub.add_parser(name, help=text)
        for o in options:
            extra = {"choices": ["fp32", "tc"]} if o.name == "mode" else {}
            sp.add_argument(o.flag, dest=o.name, type=o.kind, help=o.help, **extra)
        sp.add_argument("--config", help="JSON object of settings (flags override it)")
    return parser


def main(argv=None) -> int:
    cli_args = build_parser().parse_args(argv)
    options, run, _ = COMMANDS[cli_args.command]
    try:
        report = run(settings(options, cli_args))
    except MobaError as exc:
        print(json.dumps({"error": type(exc).__name__, "message": str(exc)}), file=sys.stderr)
        return 2
    print(report.to_json())
    return 0 if report.passed else 1


if __name__ == "__main__":
    sys.exit(main())
