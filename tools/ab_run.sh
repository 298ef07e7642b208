mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ablation.py -q -x > gpurun_out/abl_tests.log 2>&1; tail -2 gpurun_out/abl_tests.log
timeout 600 python -c "
import bench, json
r = bench.ablation_bench()
print(json.dumps([(s['stage'][:30], s['ms_per_apply'], s['marginal_speedup']) for s in r['stages']]), r['overall_speedup'])
r = bench.ablation_bench(p=4)
print(json.dumps([(s['stage'][:30], s['ms_per_apply'], s['marginal_speedup']) for s in r['stages']]), r['overall_speedup'])
"
timeout 600 python tools/abl_breakdown.py 8 2>/dev/null
