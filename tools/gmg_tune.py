"""GMG-PCG on config 3: iterations and time to 1e-8 for smoother orders / levels / coarse iterations."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2601_08374_b200.elas import GMG
P = synth.make_config(3, draw_x=False)
out = []
for levels, order, cmax in [(4, 3, 20), (4, 2, 20), (4, 4, 20), (4, 5, 20), (4, 6, 20), (4, 4, 40), (3, 4, 20), (3, 4, 60), (4, 8, 20)]:
    g = GMG.from_problem(P, levels=levels, order=order, coarse_maxit=cmax)
    b = torch.from_numpy(synth.splitmix_uniform(g.local_dofs, 11)).cuda()
    x = torch.empty_like(b)
    g.pcg(b, x, rtol=1e-8, maxit=3)
    torch.cuda.synchronize()
    t = time.perf_counter()
    it, conv, rel, _ = g.pcg(b, x, rtol=1e-8, maxit=500)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    r = dict(levels=levels, order=order, coarse_maxit=cmax, iters=it, conv=bool(conv), solve_s=round(dt, 4))
    print(json.dumps(r), flush=True)
    g.close(); del b, x; torch.cuda.empty_cache()
