"""Config-4 GDoF/s of the anisotropic operator (random SPD Voigt matrix per element) vs isotropic."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2601_08374_b200.elas import Operator
out = {}
for p in [int(a) for a in sys.argv[1:]] or range(2, 9):
    P = synth.make_config(4, p)
    x = torch.from_numpy(P.x).cuda(); y = torch.empty_like(x)
    C6 = synth.random_C6(np.random.default_rng(p), (P.nz, P.ny, P.nx))
    for name, op in (("iso", Operator.from_problem(P)), ("aniso", Operator.anisotropic(P, C6))):
        for _ in range(3): op.apply(x, y)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10): op.apply(x, y)
        b.record(); torch.cuda.synchronize()
        out[f"p{p}_{name}"] = round(P.num_dofs / (a.elapsed_time(b) / 10 / 1e3) / 1e9, 2)
        op.close(); torch.cuda.empty_cache()
    print(p, out[f"p{p}_iso"], out[f"p{p}_aniso"], flush=True)
print(json.dumps(out))
