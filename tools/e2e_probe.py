"""e2e (pinned host buffers) GDoF/s of config 5 through elas_apply_host for the lib in ELAS_LIBNAME."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2601_08374_b200.elas import Operator
P = synth.make_config(5)
op = Operator.from_problem(P)
xh = torch.from_numpy(P.x).pin_memory(); yh = torch.empty_like(xh).pin_memory()
op.apply_host(xh, yh)
t = time.perf_counter()
for _ in range(3): op.apply_host(xh, yh)
dt = (time.perf_counter() - t) / 3
print(os.environ.get("ELAS_LIBNAME", "libelas.so"), "e2e", round(P.num_dofs / dt / 1e9, 3), "GDoF/s", round(dt * 1e3, 1), "ms")
