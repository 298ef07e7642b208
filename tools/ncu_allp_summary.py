"""Summarise gpurun_out/ncu_allp_<p>.ncu-rep (tools/ncu_all_p.sh) into one JSON object per degree."""
import csv, io, json, subprocess, sys

KEYS = {"kernel": "Kernel Name", "ms": "gpu__time_duration.sum", "regs": "launch__registers_per_thread",
        "block": "launch__block_size", "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram_read": "dram__bytes_read.sum", "dram_write": "dram__bytes_write.sum",
        "smem_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "inst_executed": "smsp__inst_executed.sum", "grid": "launch__grid_size",
        "l2_hit_pct": "lts__t_sector_hit_rate.pct",
        "l1_data_pipe_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"}
out = {}
for p in range(1, 9):
    raw = subprocess.run(["ncu", "-i", f"gpurun_out/ncu_allp_{p}.ncu-rep", "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        out[str(p)] = "missing"
        continue
    hdr, units, vals = rows[0], rows[1], rows[2]
    d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))
    out[str(p)] = {k: (d.get(m, "") + (" " + u.get(m, "") if u.get(m) else "")).strip() for k, m in KEYS.items()}
    st = {}
    for h, v in d.items():   # warp-state stall samples (smsp__pcsamp_warps_issue_stalled_*)
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                st[h[len("smsp__pcsamp_warps_issue_stalled_"):]] = int(float(v.replace(",", "")))
            except ValueError:
                pass
    out[str(p)]["stalls_top"] = dict(sorted(st.items(), key=lambda kv: -kv[1])[:6])
json.dump(out, sys.stdout, indent=1)
