"""A/B: config-4 GDoF/s per p for each kernel variant named on the command line.
usage: python tools/ab_variants.py VARIANTS P...   e.g.  1,4 3 4 5"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import torch, synth
from paper_2601_08374_b200.elas import Operator
variants = [int(v) for v in sys.argv[1].split(",")]
ps = [int(a) for a in sys.argv[2:]] or list(range(1, 9))
out = {}
for p in ps:
    P = synth.make_config(4, p)
    x = torch.from_numpy(P.x).cuda(); y = torch.empty_like(x)
    for v in variants:
        try:
            op = Operator.from_problem(P, variant=v)
        except Exception as e:
            out[f"p{p}v{v}"] = str(e)[:40]; continue
        for _ in range(3): op.apply(x, y)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10): op.apply(x, y)
        b.record(); torch.cuda.synchronize()
        t = a.elapsed_time(b) / 10 / 1e3
        F = bench.alg_flops(p, P.q, P.num_elements)
        out[f"p{p}v{v}"] = (round(P.num_dofs / t / 1e9, 2), round(F / t / bench.PEAK_FP64_DERIVED, 3))
        print(p, v, out[f"p{p}v{v}"], flush=True)
        op.close(); torch.cuda.empty_cache()
    del x, y; torch.cuda.empty_cache()
print(os.environ.get("ELAS_LIBNAME", "libelas.so"), json.dumps(out))
