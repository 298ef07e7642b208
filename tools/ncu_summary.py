"""Summarise an .ncu-rep: key raw metrics, stall reasons and the top stalled SASS lines."""
import csv, io, json, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct"]
out = {}
for k in keys:
    if k in d:
        out[k] = f"{d[k]} {u.get(k, '')}".strip()
for h in hdr:
    if "dmma" in h.lower() and "pct" in h and h not in out:
        out[h] = d[h]
stall = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(float(v)) for h, v in zip(hdr, vals)
         if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued") and v}
out["stalls"] = dict(sorted(stall.items(), key=lambda kv: -kv[1])[:12])
print(json.dumps(out, indent=1))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
h2 = srows[1]
iS, iSrc = h2.index("Warp Stall Sampling (All Samples)"), h2.index("Source")
data = [r for r in srows[2:] if len(r) > iS and r[iS].isdigit()]
for r in sorted(data, key=lambda r: -int(r[iS]))[:top]:
    print(r[iS], r[0][-5:], r[iSrc][:90])
