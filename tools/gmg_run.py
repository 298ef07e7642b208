"""A few GMG-PCG iterations on config 3 (for launch-list profiling)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2601_08374_b200.elas import GMG
P = synth.make_config(3, draw_x=False)
g = GMG.from_problem(P, levels=int(os.environ.get("LEVELS", "4")), coarse_maxit=int(os.environ.get("CMAX", "30")))
b = torch.from_numpy(synth.splitmix_uniform(g.local_dofs, 11)).cuda()
x = torch.empty_like(b)
g.pcg(b, x, rtol=1e-8, maxit=3)
torch.cuda.synchronize()
t = time.perf_counter()
it, conv, rel, _ = g.pcg(b, x, rtol=1e-8, maxit=int(os.environ.get("MAXIT", "500")))
torch.cuda.synchronize()
dt = time.perf_counter() - t
print("levels", g.levels, "iters", it, conv, "ms/iter", round(dt / it * 1e3, 3))
