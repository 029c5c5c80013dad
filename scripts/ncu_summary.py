"""Summarise ncu captures (gpurun_out/*.ncu-rep, launches.csv) into profiles/.

usage: python scripts/ncu_summary.py <round-tag> [workload key, e.g. b2h16_n65536_d64]
writes profiles/<tag>_ncu_summary.md, profiles/<tag>_launches.md and
profiles/ncu_traffic.json (dram bytes per launch of each profiled stage,
read by bench.py for roofline.traffic).
"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % active"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]
STAGE_OF = {"moba_bwd": "bwd", "moba_fwd": "fwd", "route_tc_kernel": "route", "combine": "combine", "bwd_preprocess": "bwd_pre", "varlen": "varlen",
            "centroid": "centroid"}


def to_bytes(val, unit):
    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(val.replace(",", "")) * mul


def main(tag, workload=None):
    os.makedirs(PROF, exist_ok=True)
    lines = [f"# ncu summary — {tag}", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
             "(scripts/ncu_profile.sh, bench.py --steps 2 --warmup 3). Per-launch values; ncu replays "
             "each kernel, so durations are cold-cache and serialised.", ""]
    traffic = {}
    tp = os.path.join(PROF, "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp))
    if workload:
        traffic = {"workload": workload,
                   "source": f"profiles/{tag}_ncu_summary.md (dram__bytes_read.sum + dram__bytes_write.sum per launch)"}
    for rep in sorted(glob.glob(os.path.join(OUT, "prof_*.ncu-rep"))):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            continue
        h, u, v = rows[0], rows[1], rows[2]
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else os.path.basename(rep)
        lines += [f"## `{name[:120]}`", "", "| metric | value |", "|---|---|"]
        vals = {}
        for m, label in METRICS:
            if m in h:
                i = h.index(m)
                vals[m] = (v[i], u[i])
                lines.append(f"| {label} (`{m}`) | {v[i]} {u[i]} |")
        lines.append("")
        if "dram__bytes_read.sum" in vals:
            tb = to_bytes(*vals["dram__bytes_read.sum"]) + to_bytes(*vals["dram__bytes_write.sum"])
            for key, stage in STAGE_OF.items():
                if key in name:
                    traffic[stage] = tb
    with open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(tp, "w") as f:
        json.dump(traffic, f, indent=1)
    lc = os.path.join(OUT, "launches.csv")
    if os.path.exists(lc):
        txt = open(lc).read()
        txt = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
        rows = list(csv.DictReader(io.StringIO(txt)))
        agg = {}
        for r in rows:
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = r["Kernel Name"].split("(")[0][:80]
            t = float(r["Metric Value"].replace(",", "")) * (1e-3 if r.get("Metric Unit") in ("ns", "nsecond") else 1)
            a = agg.setdefault(k, [0, 0.0])
            a[0] += 1
            a[1] += t
        tot = sum(a[1] for a in agg.values()) or 1
        out = [f"# launch list — {tag}", "",
               "`ncu --metrics gpu__time_duration.sum --clock-control none` over `bench.py --steps 2 --warmup 3 "
               "--no-cpu --no-extra` (all launches of the process incl. warm-up and e2e pass; cold-cache, "
               "serialised: compare shares).", "", "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            out.append(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f}% |")
        with open(os.path.join(PROF, f"{tag}_launches.md"), "w") as f:
            f.write("\n".join(out) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01", sys.argv[2] if len(sys.argv) > 2 else None)
