"""Brief of an ncu report: key throughput metrics, stall reasons, hottest source lines.
usage: python scripts/ncu_brief.py REPORT.ncu-rep [n_lines]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for r in rows[2:]:
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w}: {r[i]} {units[i]}")
    st = [(h, r[i]) for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    st = sorted(st, key=lambda x: -float(x[1] or 0))[:8]
    print("  stalls:", ", ".join(f"{h[34:-28]}={float(v):.2f}" for h, v in st))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
lines = list(csv.reader(io.StringIO(src)))
if lines:
    h = lines[0]
    try:
        ci = h.index("Warp Stall Sampling (All Samples)")
        si = h.index("Source")
        tot = sum(float(x[ci] or 0) for x in lines[1:] if len(x) > ci)
        top = sorted(lines[1:], key=lambda x: -float(x[ci] or 0) if len(x) > ci else 0)[:nl]
        print(f"  top SASS by stall samples (total {tot:.0f}):")
        for x in top:
            print(f"   {float(x[ci]) / tot * 100:5.1f}%  {x[si][:110]}")
    except (ValueError, IndexError) as e:
        print("  (no source page)", e, h[:12])
