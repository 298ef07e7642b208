"""GPU parity of the GMG V-cycle through the C ABI against the
oracle (oracle/gmg.py): transfers vs the oracle's dense prolongation, one V-cycle vs the
oracle's V-cycle (coarse solves to near machine precision on both sides), GMG-PCG iteration
counts and mesh independence.

Tolerances: transfers are short sums (<= 1e-13 relative); a V-cycle composes smoothers and a
coarse PCG solved to 1e-14 on the GPU vs a dense direct solve in the oracle (<= 1e-9).
"""

import numpy as np
import pytest

import oracle
import synth
from oracle import gmg as ogmg

pytestmark = pytest.mark.gpu


def torch_mod():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def mesh_of(P):
    lam, mu = P.material_arrays()
    return oracle.Mesh(P.vertex_array(), P.p, P.q, lam, mu, P.dirichlet_faces)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("p,dims,faces", [(1, (4, 2, 2), 1), (2, (2, 4, 2), 1 | 8), (3, (2, 2, 4), 0),
                                          (6, (2, 2, 2), 1), (8, (2, 2, 2), 2)])
def test_transfers_vs_oracle(p, dims, faces):
    torch = torch_mod()
    from paper_2601_08374_b200.elas import GMG
    P = synth.make_problem("t", *dims, p, p + 1, perturb=True, lognormal_material=True, faces=faces, seed=p)
    g = GMG.from_problem(P, levels=2)
    fine = mesh_of(P)
    coarse = ogmg.coarsen(fine)
    Pm = ogmg.prolongation(fine, coarse)
    nf, nc = g.level_dofs(0), g.level_dofs(1)
    assert Pm.shape == (nf, nc)
    uc = synth.splitmix_uniform(nc, 1)
    uf = torch.empty(nf, dtype=torch.float64, device="cuda")
    g.transfer(0, False, torch.from_numpy(uc).cuda(), uf)
    torch.cuda.synchronize()
    assert rel(uf.cpu().numpy(), Pm @ uc) <= 1e-13
    rf = synth.splitmix_uniform(nf, 2)
    rc = torch.empty(nc, dtype=torch.float64, device="cuda")
    g.transfer(0, True, torch.from_numpy(rf).cuda(), rc)
    torch.cuda.synchronize()
    ref = Pm.T @ rf
    ref[oracle.constrained_mask(coarse)] = 0.0
    assert rel(rc.cpu().numpy(), ref) <= 1e-13
    g.close()


@pytest.mark.parametrize("p,dims,levels,faces", [(1, (4, 4, 4), 3, 1), (2, (4, 4, 2), 2, 1 | 16), (3, (2, 2, 2), 2, 1)])
def test_vcycle_vs_oracle(p, dims, levels, faces):
    torch = torch_mod()
    from paper_2601_08374_b200.elas import GMG
    P = synth.make_problem("t", *dims, p, p + 1, perturb=True, lognormal_material=True, faces=faces, seed=10 + p)
    G = ogmg.GMG(mesh_of(P), levels)
    g = GMG.from_problem(P, levels=levels, coarse_rtol=1e-15, coarse_maxit=5000)
    n = g.local_dofs
    b = synth.splitmix_uniform(n, 3)
    z_ref = G.vcycle(b.copy())
    z = torch.empty(n, dtype=torch.float64, device="cuda")
    g.apply(torch.from_numpy(b).cuda(), z)
    torch.cuda.synchronize()
    assert rel(z.cpu().numpy(), z_ref) <= 1e-9
    g.close()


def test_gmg_pcg_vs_oracle_iterations():
    torch = torch_mod()
    from paper_2601_08374_b200.elas import GMG
    P = synth.make_problem("t", 4, 4, 4, 2, 3, perturb=True, lognormal_material=True, faces=1, seed=21)
    m = mesh_of(P)
    G = ogmg.GMG(m, 3)
    b = synth.splitmix_uniform(m.num_dofs, 4)
    _, it_ref, _ = oracle.pcg(m, b, G.vcycle, 1e-8, 200, matvec=lambda v: G.levels[0].A @ v)
    g = GMG.from_problem(P, levels=3, coarse_rtol=1e-14, coarse_maxit=5000)
    x = torch.empty(m.num_dofs, dtype=torch.float64, device="cuda")
    bd = torch.from_numpy(b).cuda()
    it, conv, r, _ = g.pcg(bd, x, rtol=1e-8, maxit=200)
    assert conv and abs(it - it_ref) <= 1
    Ax = torch.empty_like(x)
    g.apply_op(x, Ax)
    assert float(torch.linalg.norm(Ax - bd) / torch.linalg.norm(bd)) <= 1e-6
    # the default fixed-length coarse solve (no host round trip) converges too
    g2 = GMG.from_problem(P, levels=3)
    it2, conv2, _, _ = g2.pcg(bd, x, rtol=1e-8, maxit=200)
    assert conv2 and it2 <= it_ref + 3
    g.close(); g2.close()


def test_vcycle_symmetric_and_zero():
    torch = torch_mod()
    from paper_2601_08374_b200.elas import GMG
    P = synth.make_problem("t", 4, 4, 4, 3, 5, perturb=True, lognormal_material=True, faces=1, seed=31)
    g = GMG.from_problem(P, levels=3, coarse_rtol=1e-15, coarse_maxit=5000)
    n = g.local_dofs
    x = torch.from_numpy(synth.splitmix_uniform(n, 5)).cuda()
    b = torch.from_numpy(synth.splitmix_uniform(n, 6)).cuda()
    Mx, Mb = torch.empty_like(x), torch.empty_like(b)
    g.apply(x, Mx)
    g.apply(b, Mb)
    a1, a2 = float(torch.dot(x, Mb)), float(torch.dot(Mx, b))
    assert abs(a1 - a2) <= 1e-9 * float(torch.linalg.norm(x) * torch.linalg.norm(Mb))
    z = torch.zeros_like(x)
    g.apply(torch.zeros_like(x), z)
    torch.cuda.synchronize()
    assert not bool(z.any())
    g.close()


def test_gmg_mesh_independent_on_gpu():
    """p = 4, 4^3 -> 8^3 -> 16^3 fine meshes with one more level each: iterations within 5."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import GMG
    its = []
    for k, m in enumerate((4, 8, 16)):
        P = synth.make_problem("t", m, m, m, 4, 6, perturb=True, lam=1.0, mu=0.5, faces=1, seed=40)
        g = GMG.from_problem(P, levels=2 + k)
        b = torch.from_numpy(synth.splitmix_uniform(g.local_dofs, 7)).cuda()
        x = torch.empty_like(b)
        it, conv, _, _ = g.pcg(b, x, rtol=1e-8, maxit=300)
        assert conv
        its.append(it)
        g.close()
    assert max(its) - min(its) <= 5, its


def test_gmg_errors():
    torch_mod()
    from paper_2601_08374_b200 import elas
    P = synth.make_problem("t", 3, 2, 2, 2, 3, seed=1)
    with pytest.raises(elas.ElasError, match="divisible"):
        elas.GMG.from_problem(P, levels=2)


def test_fp64_pcg_with_fp32_vcycle():
    """Mixed precision in the paper's solver: FP64 CG on the FP64 operator, V-cycle built from
    ELAS_VARIANT_FOLDED_F32 operators; converges to the FP64 tolerance in about the same
    number of iterations as the FP64 V-cycle."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import GMG, Operator, VARIANT_FOLDED_F32, elas_pcg_gmg
    P = synth.make_problem("t", 8, 8, 8, 3, 5, perturb=True, lognormal_material=True, faces=1, seed=55)
    op = Operator.from_problem(P)
    g64 = GMG.from_problem(P, levels=3)
    g32 = GMG.from_problem(P, levels=3, variant=VARIANT_FOLDED_F32)
    b = torch.from_numpy(synth.splitmix_uniform(op.local_dofs, 12)).cuda()
    x = torch.empty_like(b)
    it64, c64, _, _ = elas_pcg_gmg(op.h, g64.h, b, x, 1e-10, 300)
    it32, c32, r32, _ = elas_pcg_gmg(op.h, g32.h, b, x, 1e-10, 300)
    assert c64 and c32 and r32 <= 1e-10 and it32 <= it64 + 3
    Ax = torch.empty_like(b)
    op.apply(x, Ax)
    assert float(torch.linalg.norm(Ax - b) / torch.linalg.norm(b)) <= 1e-8
    g32.close(); g64.close(); op.close()


@pytest.mark.parametrize("nranks,p,levels", [(2, 2, 2), (4, 1, 3), (2, 6, 2)])
def test_slab_transfers_loopback(nranks, p, levels):
    """Z-slab GMG (external-exchange mode, P slab hierarchies on ONE GPU): prolongation is local and
    equals the single-GPU one on every slab; restriction counts a shared fine interface plane on
    the rank below only, and after the coarse interface planes are summed with the library's
    plane-add (elas_interface_add) it equals the single-GPU restriction.  The NCCL mode runs the
    same kernels with exchange_planes doing that sum."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import GMG, elas_interface_add
    f = 1 << (levels - 1)
    nz = nranks * f * 2
    P = synth.make_problem("sg", f, 2 * f, nz, p, p + 1, perturb=True, lognormal_material=True,
                           faces=1 | 16 | 32, seed=61)
    g = GMG.from_problem(P, levels=levels)
    gs = [GMG.from_problem(P, levels=levels, rank=r, nranks=nranks) for r in range(nranks)]
    rng = np.random.default_rng(5)
    for lvl in range(levels - 1):
        fo, co = g.level_op(lvl), g.level_op(lvl + 1)
        nf, nc = g.level_dofs(lvl), g.level_dofs(lvl + 1)
        Nf, Nc = nf // 3, nc // 3
        nzf, nzc = nz >> lvl, nz >> (lvl + 1)
        pf, pc = Nf // (nzf * p + 1), Nc // (nzc * p + 1)          # nodes per plane
        vf = torch.from_numpy(rng.uniform(-1, 1, nf)).cuda()
        vc = torch.from_numpy(rng.uniform(-1, 1, nc)).cuda()
        rf_full, pc_full = torch.empty(nc, dtype=torch.float64, device="cuda"), torch.empty_like(vf)
        g.transfer(lvl, True, vf, rf_full)
        g.transfer(lvl, False, vc, pc_full)
        parts, outs = [], []
        for r in range(nranks):
            zf0, zf1 = r * nzf // nranks, (r + 1) * nzf // nranks
            zc0, zc1 = r * nzc // nranks, (r + 1) * nzc // nranks
            vfl = vf.view(3, -1, pf)[:, zf0 * p:zf1 * p + 1].contiguous().reshape(-1)
            vcl = vc.view(3, -1, pc)[:, zc0 * p:zc1 * p + 1].contiguous().reshape(-1)
            assert vfl.numel() == gs[r].level_dofs(lvl) and vcl.numel() == gs[r].level_dofs(lvl + 1)
            rl = torch.empty_like(vcl)
            pl = torch.empty_like(vfl)
            gs[r].transfer(lvl, True, vfl, rl)
            gs[r].transfer(lvl, False, vcl, pl)
            torch.cuda.synchronize()
            # prolongation: local, equal to the full one on the slab
            ref = pc_full.view(3, -1, pf)[:, zf0 * p:zf1 * p + 1].reshape(-1)
            assert torch.allclose(pl, ref, rtol=0, atol=1e-13 * float(ref.abs().max()))
            parts.append((rl.view(3, -1, pc)[:, 0].contiguous(), rl.view(3, -1, pc)[:, -1].contiguous()))
            outs.append((rl, zc0, zc1))
        for r, (rl, zc0, zc1) in enumerate(outs):
            lo = parts[r - 1][1] if r > 0 else None
            hi = parts[r + 1][0] if r < nranks - 1 else None
            elas_interface_add(gs[r].level_op(lvl + 1), rl, lo, hi)
        torch.cuda.synchronize()
        for rl, zc0, zc1 in outs:
            ref = rf_full.view(3, -1, pc)[:, zc0 * p:zc1 * p + 1].reshape(-1)
            assert torch.allclose(rl, ref, rtol=0, atol=1e-13 * float(rf_full.abs().max()))
    with pytest.raises(Exception):       # the V-cycle needs NCCL in slab mode
        gs[0].apply(torch.zeros(gs[0].local_dofs, dtype=torch.float64, device="cuda"),
                    torch.zeros(gs[0].local_dofs, dtype=torch.float64, device="cuda"))
    for h in gs + [g]:
        h.close()
