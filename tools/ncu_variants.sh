#!/bin/bash
# ncu --set full of secondary kernels at config 4, p = 6 (FP32 folded, geometry on the fly, SIMT,
# tensor-core) and p = 8 (ablation +SF gradient kernel); summaries into gpurun_out/ncu_variants.json
set -u
mkdir -p gpurun_out
for spec in "6 5 apply_eo f32" "6 6 apply_eo otf" "6 1 apply_kernel simt" "6 2 apply_tc tc" "8 8 grad_sf ablsf"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none -k "regex:$3" -s 1 -c 1 -o gpurun_out/ncu_var_$4 -f \
      python tools/run_variant.py $1 $2 3 > /dev/null 2>&1
  echo "$4 rc=$?"
done
python - <<'PY'
import csv, io, json, subprocess
KEYS = {"kernel": "Kernel Name", "ms": "gpu__time_duration.sum", "regs": "launch__registers_per_thread",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "dmma_pipe_pct": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram_read": "dram__bytes_read.sum", "dram_write": "dram__bytes_write.sum",
        "smem_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"}
out = {}
for tag in ("f32", "otf", "simt", "tc", "ablsf"):
    raw = subprocess.run(["ncu", "-i", f"gpurun_out/ncu_var_{tag}.ncu-rep", "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        out[tag] = "missing"; continue
    d, u = dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))
    out[tag] = {k: (d.get(m, "") + (" " + u.get(m, "") if u.get(m) else "")).strip() for k, m in KEYS.items()}
json.dump(out, open("gpurun_out/ncu_variants.json", "w"), indent=1)
PY
rm -f gpurun_out/ncu_var_*.ncu-rep
