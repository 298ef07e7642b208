"""Apply one kernel variant a few times on config 4 (for ncu captures): run_variant.py P VARIANT [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2601_08374_b200.elas import Operator
p, v = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
P = synth.make_config(4, p)
op = Operator.from_problem(P, variant=v)
x = torch.from_numpy(P.x).cuda(); y = torch.empty_like(x)
for _ in range(reps):
    op.apply(x, y)
torch.cuda.synchronize()
print("ok", p, v, op.variant)
