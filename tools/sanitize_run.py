"""Small applies of every variant / mode for compute-sanitizer (memcheck / racecheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2601_08374_b200.elas import Operator, GMG, PC_CHEBYSHEV
cases = [(1, 3, 3), (1, 3, 4), (1, 3, 6), (2, 4, 4), (3, 5, 4), (4, 6, 4), (5, 7, 4), (6, 8, 4), (6, 8, 2), (6, 8, 1),
         (7, 9, 4), (8, 10, 4), (4, 6, 5), (6, 8, 5), (2, 4, 6), (6, 8, 6), (8, 10, 6), (3, 4, 4), (3, 5, 1)]
for p, q, v in cases:
    P = synth.make_problem("t", 3, 2, 3, p, q, perturb=True, lognormal_material=True, faces=1 | 32, seed=p)
    op = Operator.from_problem(P, variant=v)
    x = torch.from_numpy(P.x).cuda(); y = torch.empty_like(x)
    op.apply(x, y)
    if v in (4, 5, 6):
        op.set_deterministic(True); op.apply(x, y); op.set_deterministic(False)
    d = torch.empty_like(x); op.diagonal(d)
    torch.cuda.synchronize()
    op.close()
    print("ok", p, q, v, flush=True)
P = synth.make_problem("t", 4, 4, 4, 2, 3, perturb=True, lognormal_material=True, faces=1, seed=3)
g = GMG.from_problem(P, levels=3)
b = torch.from_numpy(synth.splitmix_uniform(g.local_dofs, 1)).cuda(); x = torch.empty_like(b)
print("gmg", g.pcg(b, x, rtol=1e-6, maxit=20)[:2])
op = Operator.from_problem(P); ch = op.chebyshev(); print("pcg", op.pcg(b, x, precond=PC_CHEBYSHEV, cheb=ch, maxit=20)[:2])
xh = b.cpu().pin_memory(); yh = torch.empty_like(xh).pin_memory(); op.apply_host(xh, yh); print("host ok")
