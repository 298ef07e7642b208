import os, sys
sys.path.insert(0, "/root/repo")
import torch, synth
from paper_2601_08374_b200.elas import Operator
P = synth.make_config(4, 6)
op = Operator.from_problem(P)
op.set_deterministic(True)
x = torch.from_numpy(P.x).cuda(); y = torch.empty_like(x)
for _ in range(3): op.apply(x, y)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): op.apply(x, y)
b.record(); torch.cuda.synchronize()
print("colored p6 cfg4 GDoF/s", P.num_dofs / (a.elapsed_time(b) / 10 / 1e3) / 1e9)
