"""Per-kernel times of the ablation pipelines at config 4 (torch profiler): python tools/abl_breakdown.py P"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from torch.profiler import profile, ProfilerActivity
from paper_2601_08374_b200.elas import Operator
p = int(sys.argv[1]) if len(sys.argv) > 1 else 8
P = synth.make_config(4, p)
x = torch.from_numpy(P.x).cuda(); y = torch.empty_like(x)
for v in (7, 8, 9):
    op = Operator.from_problem(P, variant=v)
    op.apply(x, y); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        op.apply(x, y); torch.cuda.synchronize()
    ks = [(e.name.split("(")[0][-40:], e.device_time / 1e3) for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    print(v, [(n, round(t, 3)) for n, t in ks])
    op.close(); torch.cuda.empty_cache()
