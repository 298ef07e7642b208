"""GPU parity of the solver layer through the C ABI: matrix-free
diagonal, power-iteration lambda_max, Chebyshev smoother and PCG against the oracle
(oracle/solvers.py) on the same seeded inputs.

Tolerances: the diagonal is a sum of positive terms (relative max error <= 1e-12); the power
estimate, Chebyshev output and fixed-iteration PCG iterates are smooth functions of inputs that
agree to rounding (<= 1e-11 relative; PCG iterates <= 1e-10 after 8 iterations, rounding
amplified by the Krylov recurrences).
"""

import numpy as np
import pytest

import oracle
import synth

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


def gpu_diag(P, variant=0):
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    op = Operator.from_problem(P, variant=variant)
    d = torch.full((P.num_dofs,), np.nan, dtype=torch.float64, device="cuda")
    op.diagonal(d)
    torch.cuda.synchronize()
    v = op.variant
    op.close()
    return d.cpu().numpy(), v


@pytest.mark.parametrize("p", range(1, 9))
@pytest.mark.parametrize("dq", [1, 2])
def test_diagonal_vs_oracle(p, dq):
    P = synth.make_problem("t", 3, 2, 2, p, p + dq, perturb=True, lognormal_material=True,
                           faces=1 | 8 | 32, seed=300 + p)
    d_ref = oracle.diagonal(mesh_of(P))
    d, _ = gpu_diag(P)
    assert np.abs(d - d_ref).max() <= 1e-12 * np.abs(d_ref).max()


@pytest.mark.parametrize("p,q,variant", [(1, 3, 3), (1, 2, 1), (6, 8, 2), (6, 8, 4), (4, 6, 1)])
def test_diagonal_every_qdata_layout(p, q, variant):
    """E32 (thread kernel), TC6 (tensor-core kernel) and the line layout give the same diagonal."""
    P = synth.make_problem("t", 2, 3, 2, p, q, perturb=True, lognormal_material=True, faces=2, seed=7)
    d, v = gpu_diag(P, variant)
    assert v == variant
    d_ref = oracle.diagonal(mesh_of(P))
    assert np.abs(d - d_ref).max() <= 1e-12 * np.abs(d_ref).max()


def test_diagonal_config2_full():
    P = synth.make_config(2)
    d, _ = gpu_diag(P)
    d_ref = oracle.diagonal(mesh_of(P))
    assert np.abs(d - d_ref).max() <= 1e-12 * np.abs(d_ref).max()
    assert (d > 0).all()


def small_problem(p=2, faces=1, seed=11, dims=(3, 2, 3)):
    return synth.make_problem("t", *dims, p, p + 2, perturb=True, lognormal_material=True, faces=faces, seed=seed)


@pytest.mark.parametrize("p", [1, 2, 4, 6])
def test_power_iteration_and_chebyshev_vs_oracle(p):
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = small_problem(p, seed=20 + p)
    m = mesh_of(P)
    n = P.num_dofs
    v0 = synth.splitmix_uniform(n, 5)
    d_ref = oracle.diagonal(m)
    lam_ref = oracle.power_lambda_max(m, d_ref, v0, 10)
    op = Operator.from_problem(P)
    ch = op.chebyshev(order=3, alpha=0.1, beta=1.1, power_iters=10, v0=torch.from_numpy(v0).cuda())
    assert abs(ch.lambda_max - lam_ref) <= 1e-11 * lam_ref
    b = synth.splitmix_uniform(n, 6)
    x0 = synth.splitmix_uniform(n, 7)
    x_ref = oracle.chebyshev(m, d_ref, lam_ref, 3, 0.1, 1.1, b, x0)
    bd, xd = torch.from_numpy(b).cuda(), torch.from_numpy(x0).cuda()
    ch.apply(bd, xd)
    torch.cuda.synchronize()
    assert rel(xd.cpu().numpy(), x_ref) <= 1e-11
    ch.close()
    op.close()


def test_default_start_vector_is_splitmix():
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = small_problem(2, seed=31)
    op = Operator.from_problem(P)
    op.set_deterministic(True)     # atomics would make the two estimates differ in the last bit
    a = op.chebyshev(power_iters=4, seed=123).lambda_max
    v0 = torch.from_numpy(synth.splitmix_uniform(P.num_dofs, 123)).cuda()
    b = op.chebyshev(power_iters=4, v0=v0).lambda_max
    op.close()
    assert a == b


@pytest.mark.parametrize("order", [1, 2, 5])
def test_chebyshev_orders_and_fixed_point(order):
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = small_problem(3, faces=1 | 2, seed=40 + order)
    m = mesh_of(P)
    op = Operator.from_problem(P)
    ch = op.chebyshev(order=order, alpha=0.2, beta=1.0, power_iters=8, seed=1)
    d_ref = oracle.diagonal(m)
    lam_ref = oracle.power_lambda_max(m, d_ref, synth.splitmix_uniform(P.num_dofs, 1), 8)
    b = synth.splitmix_uniform(P.num_dofs, 2)
    x0 = np.zeros(P.num_dofs)
    x_ref = oracle.chebyshev(m, d_ref, lam_ref, order, 0.2, 1.0, b, x0)
    xd = torch.zeros(P.num_dofs, dtype=torch.float64, device="cuda")
    ch.apply(torch.from_numpy(b).cuda(), xd)
    torch.cuda.synchronize()
    assert rel(xd.cpu().numpy(), x_ref) <= 1e-11
    # b = A x exactly -> x unchanged
    xs = torch.from_numpy(synth.splitmix_uniform(P.num_dofs, 3)).cuda()
    bs = torch.empty_like(xs)
    op.apply(xs, bs)
    x2 = xs.clone()
    ch.apply(bs, x2)
    torch.cuda.synchronize()
    assert float(torch.linalg.norm(x2 - xs) / torch.linalg.norm(xs)) <= 1e-13
    ch.close()
    op.close()


@pytest.mark.parametrize("prec", ["none", "jacobi", "cheb"])
def test_pcg_fixed_iterations_vs_oracle(prec):
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator, PC_NONE, PC_JACOBI, PC_CHEBYSHEV
    P = small_problem(2, faces=1, seed=50, dims=(4, 3, 3))
    m = mesh_of(P)
    n = P.num_dofs
    b = synth.splitmix_uniform(n, 8)
    d_ref = oracle.diagonal(m)
    lam_ref = oracle.power_lambda_max(m, d_ref, synth.splitmix_uniform(n, 9), 10)
    M = {"none": None, "jacobi": lambda r: r / d_ref,
         "cheb": lambda r: oracle.chebyshev(m, d_ref, lam_ref, 3, 0.1, 1.1, r, np.zeros_like(r))}[prec]
    K = 8   # finite-precision CG iterates drift apart with K (rounding amplified by the Krylov
            # recurrences: 1.7e-8 after 25 unpreconditioned iterations); 8 keeps it at rounding level
    x_ref, it_ref, hist_ref = oracle.pcg(m, b, M, 0.0, K)
    op = Operator.from_problem(P)
    ch = op.chebyshev(power_iters=10, seed=9) if prec == "cheb" else None
    pc = {"none": PC_NONE, "jacobi": PC_JACOBI, "cheb": PC_CHEBYSHEV}[prec]
    xd = torch.empty(n, dtype=torch.float64, device="cuda")
    it, conv, relres, hist = op.pcg(torch.from_numpy(b).cuda(), xd, precond=pc, cheb=ch, rtol=0.0, maxit=K, history=True)
    assert it == K == it_ref
    assert rel(xd.cpu().numpy(), x_ref) <= 1e-10
    assert np.abs(hist - np.array(hist_ref)).max() <= 1e-10
    if ch is not None:
        ch.close()
    op.close()


def test_pcg_converges_and_zero_rhs():
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator, PC_JACOBI, PC_CHEBYSHEV
    P = small_problem(4, faces=1, seed=60, dims=(4, 4, 4))
    n = P.num_dofs
    op = Operator.from_problem(P)
    b = torch.from_numpy(synth.splitmix_uniform(n, 10)).cuda()
    x = torch.empty_like(b)
    it_j, conv_j, r_j, _ = op.pcg(b, x, precond=PC_JACOBI, rtol=1e-8, maxit=5000)
    assert conv_j and r_j <= 1e-8
    Ax = torch.empty_like(b)
    op.apply(x, Ax)
    assert float(torch.linalg.norm(Ax - b) / torch.linalg.norm(b)) <= 1e-6
    ch = op.chebyshev(power_iters=10, seed=3)
    it_c, conv_c, r_c, _ = op.pcg(b, x, precond=PC_CHEBYSHEV, cheb=ch, rtol=1e-8, maxit=5000)
    assert conv_c and it_c < it_j
    z = torch.zeros_like(b)
    it0, conv0, _, _ = op.pcg(z, x, precond=PC_JACOBI, rtol=1e-8, maxit=10)
    assert it0 == 0 and conv0 and not bool(x.any())
    ch.close()
    op.close()


def test_solver_error_paths():
    torch = torch_mod()
    from paper_2601_08374_b200 import elas
    P = small_problem(2, seed=70, dims=(2, 2, 4))
    op = elas.Operator.from_problem(P)
    b = torch.zeros(P.num_dofs, dtype=torch.float64, device="cuda")
    with pytest.raises(elas.ElasError, match="Chebyshev"):
        op.pcg(b, b.clone(), precond=elas.PC_CHEBYSHEV, cheb=None)
    with pytest.raises(elas.ElasError, match="alpha"):
        op.chebyshev(alpha=0.5, beta=0.4)
    op2 = elas.Operator.from_problem(P, rank=0, nranks=2)
    with pytest.raises(elas.ElasError, match="NCCL slab mode"):
        op2.chebyshev()
    op2.close()
    op.close()


def test_pcg_fp64_with_fp32_chebyshev():
    """Mixed precision in the solver: FP64 PCG (FP64 operator) preconditioned by a Chebyshev
    smoother built on the FP32 operator of the same mesh converges to the FP64 tolerance."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator, PC_CHEBYSHEV, VARIANT_FOLDED_F32
    P = small_problem(4, faces=1, seed=61, dims=(4, 4, 4))
    n = P.num_dofs
    op = Operator.from_problem(P)
    op32 = Operator.from_problem(P, variant=VARIANT_FOLDED_F32)
    ch64 = op.chebyshev(power_iters=10, seed=3)
    ch32 = op32.chebyshev(power_iters=10, seed=3)
    assert abs(ch32.lambda_max - ch64.lambda_max) <= 1e-5 * ch64.lambda_max
    b = torch.from_numpy(synth.splitmix_uniform(n, 10)).cuda()
    x = torch.empty_like(b)
    it64, c64, _, _ = op.pcg(b, x, precond=PC_CHEBYSHEV, cheb=ch64, rtol=1e-10, maxit=3000)
    it32, c32, r32, _ = op.pcg(b, x, precond=PC_CHEBYSHEV, cheb=ch32, rtol=1e-10, maxit=3000)
    assert c64 and c32 and r32 <= 1e-10
    assert it32 <= int(1.2 * it64) + 2
    Ax = torch.empty_like(b)
    op.apply(x, Ax)
    assert float(torch.linalg.norm(Ax - b) / torch.linalg.norm(b)) <= 1e-7
    ch32.close(); ch64.close(); op32.close(); op.close()


@pytest.mark.parametrize("nranks", [2, 3, 5])
def test_distributed_dot_ownership(nranks):
    """elas_dot on slab operators counts every replicated interface plane once: the sum of the
    rank-local partials (external-exchange mode, one GPU) equals the single-operator dot."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator, elas_dot
    P = synth.make_problem("t", 3, 2, 10, 3, 5, perturb=True, seed=70 + nranks)
    n = P.num_dofs
    a = synth.splitmix_uniform(n, 1)
    b = synth.splitmix_uniform(n, 2)
    op = Operator.from_problem(P)
    full = elas_dot(op.h, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    op.close()
    assert abs(full - float(a @ b)) <= 1e-12 * abs(float(np.abs(a) @ np.abs(b)))
    Nx, Ny, Nz = P.node_dims
    ag, bg = a.reshape(3, Nz, Ny * Nx), b.reshape(3, Nz, Ny * Nx)
    tot = 0.0
    for r in range(nranks):
        o = Operator.from_problem(P, rank=r, nranks=nranks)
        z0, z1 = o.zrange
        al = torch.from_numpy(np.ascontiguousarray(ag[:, z0 * P.p:z1 * P.p + 1])).cuda().reshape(-1)
        bl = torch.from_numpy(np.ascontiguousarray(bg[:, z0 * P.p:z1 * P.p + 1])).cuda().reshape(-1)
        tot += elas_dot(o.h, al, bl)
        o.close()
    assert abs(tot - full) <= 1e-12 * abs(float(np.abs(a) @ np.abs(b)))
