"""Config-5 (bench workload) apply timing for the library named by ELAS_LIBNAME (no bench extras)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2601_08374_b200.elas import Operator
P = synth.make_config(5)
op = Operator.from_problem(P)
x = torch.from_numpy(P.x).cuda(); y = torch.empty_like(x)
for _ in range(3): op.apply(x, y)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): op.apply(x, y)
b.record(); torch.cuda.synchronize()
t = a.elapsed_time(b) / 10 / 1e3
print(os.environ.get("ELAS_LIBNAME", "libelas.so"), "cfg5", round(P.num_dofs / t / 1e9, 3), "GDoF/s")
