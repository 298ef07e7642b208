"""Quick tuning sweep: config-4 GDoF/s per p for the library named by ELAS_LIBNAME."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
VAR = int(os.environ.get("ELAS_VARIANT", "0"))
ps = [int(a) for a in sys.argv[1:]] or list(range(1, 9))
out = {}
import torch, synth
from paper_2601_08374_b200.elas import Operator, elas_profile, elas_profile_read
for p in ps:
    P = synth.make_config(4, p)
    op = Operator.from_problem(P, variant=VAR if (VAR != 2 or p == 6) else 0)
    x = torch.from_numpy(P.x).cuda(); y = torch.empty_like(x)
    for _ in range(3): op.apply(x, y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): op.apply(x, y)
    b.record(); torch.cuda.synchronize()
    t = a.elapsed_time(b) / 10 / 1e3
    F = bench.alg_flops(p, P.q, P.num_elements)
    out[p] = (round(P.num_dofs / t / 1e9, 2), round(F / t / bench.PEAK_FP64_DERIVED, 3))
    op.close(); del x, y; torch.cuda.empty_cache()
print(os.environ.get("ELAS_LIBNAME", "libelas.so"), "variant", VAR, json.dumps(out))
