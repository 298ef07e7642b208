"""Config 5 (683M dofs): GDoF/s of each kernel variant named on the command line (e.g. 2,4)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2601_08374_b200.elas import Operator
P = synth.make_config(5)
x = torch.from_numpy(P.x).cuda(); y = torch.empty_like(x)
for v in [int(a) for a in sys.argv[1].split(",")]:
    op = Operator.from_problem(P, variant=v)
    for _ in range(3): op.apply(x, y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): op.apply(x, y)
    b.record(); torch.cuda.synchronize()
    t = a.elapsed_time(b) / 10 / 1e3
    print("cfg5 variant", v, round(P.num_dofs / t / 1e9, 2), "GDoF/s", flush=True)
    op.close(); torch.cuda.empty_cache()
