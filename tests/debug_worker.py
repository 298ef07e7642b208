"""Runs under ELAS_LIBNAME=libelas_debug.so (tests/test_gpu_debug.py): every kernel family on
small meshes with Dirichlet faces and ragged element counts, parity vs the oracle, and zero failed
device bounds checks (the compute-sanitizer stand-in).  Prints "DEBUG OK <n>"."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import oracle
import synth
from paper_2601_08374_b200 import elas
from paper_2601_08374_b200.elas import Operator


def ref(P):
    lam, mu = P.material_arrays()
    return oracle.apply(oracle.Mesh(P.vertex_array(), P.p, P.q, lam, mu, P.dirichlet_faces), P.x)


def run(P, **kw):
    det = kw.pop("deterministic", False)
    op = Operator.from_problem(P, **kw)
    if det:
        op.set_deterministic(True)
    x = torch.from_numpy(P.x).cuda()
    y = torch.full_like(x, float("nan"))
    op.apply(x, y)
    torch.cuda.synchronize()
    op.close()
    return y.cpu().numpy()


def main():
    assert elas.elas_debug_build(), "not the debug library"
    n, line = elas.elas_debug_checks(selftest=True)
    assert n >= 1 and line > 0, (n, line)           # the checks are live
    assert elas.elas_debug_checks()[0] == 0          # and were reset
    cases = [(synth.make_config(1), {}), (synth.make_config(2), {})]
    for p in range(1, 9):
        cases.append((synth.make_problem("d", 3, 2, 3, p, p + 2, perturb=True, lognormal_material=True,
                                         faces=1 | 8 | 32, seed=200 + p), {}))
    P6 = synth.make_problem("d6", 2, 3, 2, 6, 8, perturb=True, lognormal_material=True, faces=2 | 16, seed=7)
    cases += [(P6, {"variant": elas.VARIANT_SIMT}), (P6, {"variant": elas.VARIANT_TENSOR}),
              (synth.make_problem("d1", 5, 3, 2, 1, 2, perturb=True, faces=63, seed=8), {"variant": elas.VARIANT_THREAD}),
              (synth.make_problem("do", 3, 3, 2, 3, 5, perturb=True, lognormal_material=True, faces=1, seed=9),
               {"variant": elas.VARIANT_FOLDED_OTF}),
              (synth.make_problem("dc", 3, 2, 4, 4, 6, perturb=True, lognormal_material=True, faces=4 | 32, seed=10),
               {"deterministic": True})]
    for P, kw in cases:
        y = run(P, **dict(kw))
        y_ref = ref(P)
        err = float(np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref))
        assert err <= 1e-12, (P.name, P.p, kw, err)
    n, line = elas.elas_debug_checks()
    assert n == 0, f"{n} failed device bounds checks, first at line {line}"
    print(f"DEBUG OK {len(cases)}", flush=True)


if __name__ == "__main__":
    main()
