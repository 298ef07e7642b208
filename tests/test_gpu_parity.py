"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Tolerance: relative L2 error <= 1e-12 over all dofs, or over the sampled rows at full size
(north_star, BASELINE.json).  Near-zero outputs (rigid modes) use the
scaled absolute form ||A r|| <= tol ||A||_est ||r||.
"""

import numpy as np
import pytest

import oracle
import synth
from tests import oracle_pool

pytestmark = pytest.mark.gpu

TOL = 1e-12


def torch_mod():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def oracle_mesh(P):
    lam, mu = P.material_arrays()
    return oracle.Mesh(P.vertex_array(), P.p, P.q, lam, mu, P.dirichlet_faces)


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def gpu_apply(P, x=None, op=None):
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    own = op is None
    if own:
        op = Operator.from_problem(P)
    xd = torch.from_numpy(np.ascontiguousarray(P.x if x is None else x)).cuda()
    yd = torch.full_like(xd, np.nan)
    op.apply(xd, yd)
    torch.cuda.synchronize()
    y = yd.cpu().numpy()
    if own:
        op.close()
    return y


def sample_rows(P, n, seed, extra=()):
    rng = np.random.default_rng(seed)
    rows = rng.choice(P.num_dofs, size=min(n, P.num_dofs), replace=False)
    return np.unique(np.concatenate([rows, np.asarray(extra, dtype=np.int64)]))


def plane_rows(P, K, count, seed):
    """Rows on global node plane K (all three components), sampled."""
    Nx, Ny, Nz = P.node_dims
    N = Nx * Ny * Nz
    rng = np.random.default_rng(seed)
    idx = rng.choice(Nx * Ny, size=min(count, Nx * Ny), replace=False)
    return np.concatenate([c * N + K * Nx * Ny + idx for c in range(3)])


# ---------------------------------------------------------------------------------------

def test_config1_full_and_brute_force():
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = synth.make_config(1)
    m = oracle_mesh(P)
    y_ref = oracle.apply(m, P.x)
    y = gpu_apply(P)
    assert rel_l2(y, y_ref) <= TOL
    # brute force: the GPU operator applied to all 375 unit vectors equals the oracle's A
    A_ref = oracle.assemble_dense(m)
    op = Operator.from_problem(P)
    n = P.num_dofs
    cols = np.zeros((n, n))
    I = torch.eye(n, dtype=torch.float64, device="cuda")
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    for j in range(n):
        op.apply(I[j].contiguous(), out)
        cols[:, j] = out.cpu().numpy()
    op.close()
    assert np.abs(cols - A_ref).max() <= 1e-13 * np.abs(A_ref).max()


@pytest.mark.parametrize("p", range(1, 9))
@pytest.mark.parametrize("dq", [1, 2])
def test_all_degrees_small_mesh(p, dq):
    """Perturbed trilinear geometry, per-element material, three Dirichlet faces, a ragged
    element count (3x2x3 = 18 elements: several CTAs plus a partial one for every p)."""
    P = synth.make_problem("t", 3, 2, 3, p, p + dq, perturb=True, lognormal_material=True,
                           faces=synth.FACE_XMIN | 8 | 16, seed=100 + p)
    y_ref = oracle.apply(oracle_mesh(P), P.x)
    y = gpu_apply(P)
    assert rel_l2(y, y_ref) <= TOL


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_many_ctas_ragged(p):
    """More elements than one wave of CTAs per... and a count that is not a multiple of EB."""
    P = synth.make_problem("t", 7, 5, 3, p, p + 2, lengths=(1.4, 1.0, 0.6), perturb=True,
                           lognormal_material=True, faces=2 | 4, seed=7 + p)
    y_ref = oracle.apply(oracle_mesh(P), P.x)
    assert rel_l2(gpu_apply(P), y_ref) <= TOL


@pytest.mark.parametrize("p", range(1, 9))
def test_single_element(p):
    P = synth.make_problem("t", 1, 1, 1, p, p + 2, perturb=True, lam=0.3, mu=2.0, seed=3)
    assert rel_l2(gpu_apply(P), oracle.apply(oracle_mesh(P), P.x)) <= TOL


def test_config2_full():
    P = synth.make_config(2)
    y_ref = oracle.apply(oracle_mesh(P), P.x)
    assert rel_l2(gpu_apply(P), y_ref) <= TOL


def test_config3_sampled_rows():
    """>= 4096 seeded random rows + rows on the Dirichlet face x = 0 and on an
    element-boundary plane."""
    P = synth.make_config(3)
    Nx, Ny, Nz = P.node_dims
    N = Nx * Ny * Nz
    face = np.arange(0, N, Nx)[:50]
    rows = sample_rows(P, 4096, 0, extra=np.concatenate([face, N + face, plane_rows(P, 6, 40, 1)]))
    assert rows.size >= 4096
    y = gpu_apply(P)
    y_ref = oracle_pool.apply_rows(oracle_mesh(P), P.x, rows)
    assert rel_l2(y[rows], y_ref) <= TOL
    Z = oracle.constrained_mask(oracle_mesh(P))
    assert np.array_equal(y[Z], P.x[Z])             # identity rows, bitwise


@pytest.mark.parametrize("p", range(1, 9))
def test_config4_full_size(p):
    """Full-size config 4 (~50M dofs) in the bench's launch configuration: sampled rows vs the
    oracle, plus rigid-mode and symmetry properties that hold at any size."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = synth.make_config(4, p)
    op = Operator.from_problem(P)
    x = torch.from_numpy(P.x).cuda()
    y = torch.empty_like(x)
    op.apply(x, y)
    torch.cuda.synchronize()
    yh = y.cpu().numpy()
    rows = sample_rows(P, 4096, p, extra=plane_rows(P, P.p * 3, 16, p))
    assert rows.size >= 4096
    y_ref = oracle_pool.apply_rows(oracle_mesh(P), P.x, rows)
    assert rel_l2(yh[rows], y_ref) <= TOL
    # rigid modes at full size: translation and the rotation (-y, x, 0) of the affine grid
    Nx, Ny, Nz = P.node_dims
    nodes = oracle.rules.gll_nodes(p)
    def coords(n_el, L):
        h = L / n_el
        return np.concatenate([e * h + h * nodes[:-1] for e in range(n_el)] + [[L]])
    X = torch.from_numpy(coords(P.nx, 1.0)).cuda()
    Y = torch.from_numpy(coords(P.ny, 1.0)).cuda()
    N = Nx * Ny * Nz
    r = torch.zeros(3 * N, dtype=torch.float64, device="cuda")
    r.view(3, Nz, Ny, Nx)[0] = -Y.view(1, Ny, 1)
    r.view(3, Nz, Ny, Nx)[1] = X.view(1, 1, Nx)
    Ar = torch.empty_like(r)
    op.apply(r, Ar)
    norm_est = float(torch.linalg.norm(y) / torch.linalg.norm(x))   # lower bound of ||A||
    assert float(torch.linalg.norm(Ar)) <= 1e-11 * norm_est * float(torch.linalg.norm(r))
    # symmetry x^T A z = z^T A x with a second random vector
    z = torch.rand_like(x) - 0.5
    Az = torch.empty_like(z)
    op.apply(z, Az)
    a, b = float(torch.dot(x, Az)), float(torch.dot(z, y))
    assert abs(a - b) <= 1e-12 * float(torch.linalg.norm(x) * torch.linalg.norm(Az))
    op.close()


def test_config5_full_size_sampled():
    """Config 5 (683M dofs) on one GPU in the bench's launch configuration: >= 4096 seeded random
    rows, EVERY row of the 2-GPU interface plane and sampled rows of the other 4/8-GPU
    interface planes; then the host-buffer apply (elas_apply_host, the bench's
    e2e call, 64 z-chunks) equal to the device apply."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = synth.make_config(5)
    p = P.p
    Nx, Ny, Nz = P.node_dims
    N = Nx * Ny * Nz
    K2 = (P.nz // 2) * p                                   # the P = 2 interface plane
    full_plane = np.concatenate([c * N + K2 * Nx * Ny + np.arange(Nx * Ny) for c in range(3)])
    extra = [full_plane]
    for nr in (4, 8):
        for r in range(1, nr):
            K = (r * P.nz // nr) * p
            if K != K2:
                extra.append(plane_rows(P, K, 64, 10 * nr + r))
    rows = sample_rows(P, 4096, 5, extra=np.concatenate(extra))
    assert rows.size >= 4096 + full_plane.size
    op = Operator.from_problem(P)
    y = gpu_apply(P, op=op)
    y_ref = oracle_pool.apply_rows(oracle_mesh(P), P.x, rows)
    assert rel_l2(y[rows], y_ref) <= TOL
    assert rel_l2(y[full_plane], y_ref[np.searchsorted(rows, full_plane)]) <= TOL
    # elas_apply_host at the bench's schedule (ELAS_HOST_CHUNKS = 64 z-chunks)
    xh = torch.from_numpy(P.x).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    op.apply_host(xh, yh)
    op.close()
    assert rel_l2(yh.numpy(), y) <= 1e-15
    del xh, yh


# ---------------------------------------------------------------------------------------
# semantics, edge cases and error paths
# ---------------------------------------------------------------------------------------

def test_dirichlet_identity_and_zero():
    torch = torch_mod()
    P = synth.make_problem("t", 2, 3, 2, 3, 5, perturb=True, lognormal_material=True, faces=63, seed=1)
    m = oracle_mesh(P)
    Z = oracle.constrained_mask(m)
    e = np.zeros(P.num_dofs)
    idx = np.flatnonzero(Z)[17]
    e[idx] = 1.0
    assert np.array_equal(gpu_apply(P, e), e)
    assert np.array_equal(gpu_apply(P, np.zeros(P.num_dofs)), np.zeros(P.num_dofs))


def test_apply_host_matches_device():
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = synth.make_problem("t", 4, 3, 5, 4, 6, perturb=True, lognormal_material=True, faces=1, seed=2)
    op = Operator.from_problem(P)
    yh = np.empty_like(P.x)
    op.apply_host(P.x, yh)
    yd = gpu_apply(P, op=op)
    op.close()
    assert rel_l2(yh, yd) <= 1e-15
    assert rel_l2(yh, oracle.apply(oracle_mesh(P), P.x)) <= TOL


def test_nondefault_stream():
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = synth.make_problem("t", 3, 3, 3, 2, 4, perturb=True, seed=4)
    s = torch.cuda.Stream()
    op = Operator.from_problem(P, stream=s)
    x = torch.from_numpy(P.x).cuda()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        y = torch.empty_like(x)
        op.apply(x, y)
    s.synchronize()
    assert rel_l2(y.cpu().numpy(), oracle.apply(oracle_mesh(P), P.x)) <= TOL
    op.close()


def test_error_paths_on_gpu():
    torch = torch_mod()
    from paper_2601_08374_b200 import elas
    P = synth.make_problem("t", 2, 2, 2, 2, 4, seed=1)
    V = P.vertex_array().copy()
    V[1, 1, 1] = V[0, 0, 0] - 0.1                  # invert elements around the centre vertex
    with pytest.raises(elas.ElasError, match="det J"):
        elas.elas_create(2, 2, 2, 2, 4, 1.0, 1.0, vertices=V)
    op = elas.Operator.from_problem(P)
    x = torch.from_numpy(P.x).cuda()
    with pytest.raises(elas.ElasError, match="alias"):
        op.apply(x, x)
    y = torch.empty(P.num_dofs + 1, dtype=torch.float64, device="cuda")
    with pytest.raises(elas.ElasError, match="aligned"):
        op.apply(x, y.data_ptr() + 4)
    with pytest.raises(elas.ElasError, match="external"):
        op.interface_add(y, None, None)
    op.close()


_LOOPBACK_REF = {}


def loopback_problem():
    P = synth.make_problem("t", 5, 4, 16, 6, 8, perturb=True, lognormal_material=True,
                           faces=1 | 16 | 32, seed=33)
    if "y" not in _LOOPBACK_REF:                      # one oracle apply for all partitions
        _LOOPBACK_REF["y"] = oracle.apply(oracle_mesh(P), P.x)
    return P, _LOOPBACK_REF["y"]


@pytest.mark.parametrize("nranks", [2, 3, 4, 8])
def test_slab_loopback_external_exchange(nranks):
    """P slab operators on ONE GPU in external-exchange mode, interface planes summed with the
    library's own plane-add kernel (the A6 interface sum, PAPER.md:169 P^T): equals the oracle's
    apply to 1e-12 and the single-GPU apply to 1e-14 relative."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P, y_ref = loopback_problem()
    y_full = gpu_apply(P)
    Nx, Ny, Nz = P.node_dims
    plane = Nx * Ny
    xg = P.x.reshape(3, Nz, Ny, Nx)
    ops, ys, ks = [], [], []
    for r in range(nranks):
        op = Operator.from_problem(P, rank=r, nranks=nranks)
        b, e = op.zrange
        K0, K1 = b * P.p, e * P.p
        xl = torch.from_numpy(np.ascontiguousarray(xg[:, K0:K1 + 1])).cuda().reshape(-1)
        assert xl.numel() == op.local_dofs
        yl = torch.empty_like(xl)
        op.apply(xl, yl)
        ops.append(op)
        ys.append(yl)
        ks.append((K0, K1))
    torch.cuda.synchronize()
    # partial planes (copies taken before any add)
    lo_part = [y.view(3, -1, plane)[:, 0].contiguous() for y in ys]
    hi_part = [y.view(3, -1, plane)[:, -1].contiguous() for y in ys]
    for r in range(nranks):
        lo = hi_part[r - 1] if r > 0 else None
        hi = lo_part[r + 1] if r < nranks - 1 else None
        ops[r].interface_add(ys[r], lo, hi)
    torch.cuda.synchronize()
    yg = np.empty((3, Nz, plane))
    for r in range(nranks):
        K0, K1 = ks[r]
        yg[:, K0:K1 + 1] = ys[r].view(3, -1, plane).cpu().numpy()
        if r > 0:   # replicated interface planes are bitwise equal on both sides
            assert np.array_equal(ys[r].view(3, -1, plane)[:, 0].cpu().numpy(),
                                  ys[r - 1].view(3, -1, plane)[:, -1].cpu().numpy())
    for op in ops:
        op.close()
    assert rel_l2(yg.reshape(-1), y_full) <= 1e-14
    assert rel_l2(yg.reshape(-1), y_ref) <= TOL


# ---------------------------------------------------------------------------------------
# kernel variants: FP64 tensor-core (DMMA) kernel for p = 6, q = 8 vs the SIMT kernel
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("variant", [1, 2])
@pytest.mark.parametrize("dims,faces", [((3, 2, 3), 1 | 8 | 16), ((7, 1, 2), 63), ((1, 1, 1), 0), ((4, 3, 5), 2)])
def test_p6_variants_vs_oracle(variant, dims, faces):
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = synth.make_problem("t", *dims, 6, 8, perturb=True, lognormal_material=True, faces=faces, seed=50 + variant)
    op = Operator.from_problem(P, variant=variant)
    assert op.variant == variant
    y = gpu_apply(P, op=op)
    op.close()
    assert rel_l2(y, oracle.apply(oracle_mesh(P), P.x)) <= TOL


def test_p6_variants_agree_at_config3():
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = synth.make_config(3)
    ys = []
    for variant in (1, 2):
        op = Operator.from_problem(P, variant=variant)
        ys.append(gpu_apply(P, op=op))
        op.close()
    assert rel_l2(ys[1], ys[0]) <= 1e-14


def test_tensor_variant_only_for_p6_q8():
    torch_mod()
    from paper_2601_08374_b200 import elas
    with pytest.raises(elas.ElasError, match="tensor-core"):
        elas.elas_create_ex(2, 2, 2, 4, 6, 1.0, 1.0, variant=elas.VARIANT_TENSOR)
    h = elas.elas_create_ex(2, 2, 2, 6, 8, 1.0, 1.0, variant=elas.VARIANT_TENSOR)
    assert elas.elas_variant(h) == elas.VARIANT_TENSOR
    elas.elas_destroy(h)
    h = elas.elas_create_ex(2, 2, 2, 6, 7, 1.0, 1.0)
    assert elas.elas_variant(h) == elas.VARIANT_FOLDED
    elas.elas_destroy(h)


@pytest.mark.parametrize("variant", [1, 3])
@pytest.mark.parametrize("q", [2, 3])
@pytest.mark.parametrize("dims,faces", [((5, 3, 4), 1 | 8 | 16), ((33, 2, 3), 63), ((1, 1, 1), 0), ((70, 1, 1), 2)])
def test_p1_variants_vs_oracle(variant, q, dims, faces):
    """p = 1: the one-thread-per-element kernel (and the fibre kernel) vs the oracle; element
    counts straddle the 32-element qdata blocks and the 128-thread CTAs."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = synth.make_problem("t", *dims, 1, q, perturb=True, lognormal_material=True, faces=faces, seed=60 + q)
    op = Operator.from_problem(P, variant=variant)
    assert op.variant == variant
    y = gpu_apply(P, op=op)
    op.close()
    assert rel_l2(y, oracle.apply(oracle_mesh(P), P.x)) <= TOL


# ---------------------------------------------------------------------------------------
# folded SIMT variant (even-odd folded 1D contractions), every p and both q
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("p", range(1, 9))
@pytest.mark.parametrize("dq", [1, 2])
@pytest.mark.parametrize("dims,faces", [((3, 2, 3), 1 | 8 | 16), ((1, 1, 1), 0), ((5, 4, 3), 63 ^ 16)])
def test_folded_variant_vs_oracle(p, dq, dims, faces):
    """Odd and even n and q (mid rows/columns of the folded tables), Dirichlet faces on both
    ends of a fold (nodes i and n-1-i), ragged element counts."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator, VARIANT_FOLDED
    P = synth.make_problem("t", *dims, p, p + dq, perturb=True, lognormal_material=True, faces=faces,
                           seed=200 + 10 * p + dq)
    op = Operator.from_problem(P, variant=VARIANT_FOLDED)
    assert op.variant == VARIANT_FOLDED
    y = gpu_apply(P, op=op)
    op.close()
    assert rel_l2(y, oracle.apply(oracle_mesh(P), P.x)) <= TOL


@pytest.mark.parametrize("cfg", [2, 3])
def test_folded_agrees_with_simt(cfg):
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator, VARIANT_SIMT, VARIANT_FOLDED
    P = synth.make_config(cfg)
    ys = []
    for variant in (VARIANT_SIMT, VARIANT_FOLDED):
        op = Operator.from_problem(P, variant=variant)
        ys.append(gpu_apply(P, op=op))
        op.close()
    assert rel_l2(ys[1], ys[0]) <= 1e-14


# ---------------------------------------------------------------------------------------
# mixed precision (FP32 qdata + arithmetic, FP64 vectors and scatter): NOT the 1e-12 contract
# ---------------------------------------------------------------------------------------

TOL_F32 = 1e-5   # FP32 unit roundoff 6e-8 x O(10-100) accumulated terms


@pytest.mark.parametrize("p", range(1, 9))
@pytest.mark.parametrize("dq", [1, 2])
def test_folded_f32_vs_oracle(p, dq):
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator, VARIANT_FOLDED_F32
    P = synth.make_problem("t", 3, 2, 3, p, p + dq, perturb=True, lognormal_material=True,
                           faces=1 | 8 | 16, seed=400 + 10 * p + dq)
    op = Operator.from_problem(P, variant=VARIANT_FOLDED_F32)
    assert op.variant == VARIANT_FOLDED_F32
    y = gpu_apply(P, op=op)
    op.close()
    err = rel_l2(y, oracle.apply(oracle_mesh(P), P.x))
    assert 1e-12 < err <= TOL_F32          # genuinely FP32 (not silently FP64), within the bound


def test_folded_f32_config4_sampled():
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator, VARIANT_FOLDED_F32
    P = synth.make_config(4, 6)
    op = Operator.from_problem(P, variant=VARIANT_FOLDED_F32)
    y = gpu_apply(P, op=op)
    op.close()
    rows = sample_rows(P, 128, 6)
    assert rel_l2(y[rows], oracle.apply_rows(oracle_mesh(P), P.x, rows)) <= TOL_F32


@pytest.mark.parametrize("p,dims,faces", [(2, (3, 2, 7), 16 | 32 | 1), (6, (2, 2, 19), 0), (1, (5, 4, 33), 63)])
def test_apply_host_chunked_pipeline(p, dims, faces):
    """elas_apply_host pipelines H2D / apply / D2H over z-chunks of element layers: equal to the
    device apply (chunk-boundary planes, Dirichlet z faces, uneven chunk sizes, nz > 16 chunks)."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = synth.make_problem("t", *dims, p, p + 2, perturb=True, lognormal_material=True, faces=faces, seed=77 + p)
    op = Operator.from_problem(P)
    xh = torch.from_numpy(P.x).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    op.apply_host(xh, yh)
    yd = gpu_apply(P, op=op)
    op.close()
    assert rel_l2(yh.numpy(), yd) <= 1e-15
    assert rel_l2(yh.numpy(), oracle.apply(oracle_mesh(P), P.x)) <= TOL


# ---------------------------------------------------------------------------------------
# deterministic (colored) scatter: bitwise reproducible applies
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("p,dims,faces,variant", [(2, (3, 4, 5), 1 | 32, 4), (6, (2, 3, 3), 0, 4), (4, (1, 1, 5), 63, 4),
                                                  (3, (5, 2, 2), 8, 5), (8, (2, 2, 1), 2, 4), (1, (7, 3, 4), 16, 4)])
def test_deterministic_colored_scatter(p, dims, faces, variant):
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = synth.make_problem("t", *dims, p, p + 2, perturb=True, lognormal_material=True, faces=faces, seed=90 + p)
    ys = []
    for _ in range(2):
        op = Operator.from_problem(P, variant=variant)
        op.set_deterministic(True)
        ys.append(gpu_apply(P, op=op))
        ys.append(gpu_apply(P, op=op))
        op.close()
    assert all(np.array_equal(ys[0], v) for v in ys[1:])          # bitwise, across runs and ops
    tol = TOL if variant == 4 else TOL_F32
    assert rel_l2(ys[0], oracle.apply(oracle_mesh(P), P.x)) <= tol


def test_deterministic_config4_and_slabs():
    """Full-size config 4 p = 6 colored vs atomic (1e-14), and the colored slab loopback
    (external-exchange mode, boundary layers) equal to the colored single-GPU apply bitwise."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = synth.make_config(4, 6)
    op = Operator.from_problem(P)
    y_atomic = gpu_apply(P, op=op)
    op.set_deterministic(True)
    y_col = gpu_apply(P, op=op)
    op.close()
    assert rel_l2(y_col, y_atomic) <= 1e-14
    P = synth.make_problem("t", 3, 3, 8, 3, 5, perturb=True, lognormal_material=True, faces=1, seed=5)
    op = Operator.from_problem(P)
    op.set_deterministic(True)
    y_full = gpu_apply(P, op=op)
    op.close()
    Nx, Ny, Nz = P.node_dims
    plane = Nx * Ny
    xg = P.x.reshape(3, Nz, Ny, Nx)
    ops, ys, ks = [], [], []
    for r in range(3):
        o = Operator.from_problem(P, rank=r, nranks=3)
        o.set_deterministic(True)
        b, e = o.zrange
        xl = torch.from_numpy(np.ascontiguousarray(xg[:, b * P.p:e * P.p + 1])).cuda().reshape(-1)
        yl = torch.empty_like(xl)
        o.apply(xl, yl)
        ops.append(o); ys.append(yl); ks.append((b * P.p, e * P.p))
    torch.cuda.synchronize()
    lo = [y.view(3, -1, plane)[:, 0].contiguous() for y in ys]
    hi = [y.view(3, -1, plane)[:, -1].contiguous() for y in ys]
    for r in range(3):
        ops[r].interface_add(ys[r], hi[r - 1] if r > 0 else None, lo[r + 1] if r < 2 else None)
    torch.cuda.synchronize()
    yg = np.empty((3, Nz, plane))
    for r in range(3):
        yg[:, ks[r][0]:ks[r][1] + 1] = ys[r].view(3, -1, plane).cpu().numpy()
        ops[r].close()
    assert rel_l2(yg.reshape(-1), y_full) <= 1e-14
    assert rel_l2(yg.reshape(-1), oracle.apply(oracle_mesh(P), P.x)) <= TOL   # the A6 sum vs the oracle


def test_deterministic_only_folded():
    torch_mod()
    from paper_2601_08374_b200 import elas
    P = synth.make_problem("t", 2, 2, 2, 6, 8, seed=1)
    op = elas.Operator.from_problem(P, variant=elas.VARIANT_TENSOR)
    with pytest.raises(elas.ElasError, match="folded"):
        op.set_deterministic(True)
    op.close()


# ---------------------------------------------------------------------------------------
# geometry on the fly (no stored quadrature data)
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("p", range(1, 9))
@pytest.mark.parametrize("dq", [1, 2])
def test_folded_otf_vs_oracle(p, dq):
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator, VARIANT_FOLDED_OTF
    P = synth.make_problem("t", 3, 2, 3, p, p + dq, perturb=True, lognormal_material=True,
                           faces=1 | 8 | 16, seed=500 + 10 * p + dq)
    op = Operator.from_problem(P, variant=VARIANT_FOLDED_OTF)
    assert op.variant == VARIANT_FOLDED_OTF
    y = gpu_apply(P, op=op)
    d = torch.empty(P.num_dofs, dtype=torch.float64, device="cuda")
    op.diagonal(d)
    op.set_deterministic(True)
    y2 = gpu_apply(P, op=op)
    op.close()
    assert rel_l2(y, oracle.apply(oracle_mesh(P), P.x)) <= TOL
    assert rel_l2(y2, y) <= 1e-14
    d_ref = oracle.diagonal(oracle_mesh(P))
    assert np.abs(d.cpu().numpy() - d_ref).max() <= 1e-12 * np.abs(d_ref).max()


def test_folded_otf_config5_sampled():
    """Config 5 (683M dofs) without quadrature data: 0.3 GB of geometry instead of 38.7 GB."""
    P = synth.make_config(5)
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator, VARIANT_FOLDED_OTF
    op = Operator.from_problem(P, variant=VARIANT_FOLDED_OTF)
    y = gpu_apply(P, op=op)
    op.close()
    rows = sample_rows(P, 256, 15, extra=plane_rows(P, 128 * P.p, 8, 3))
    assert rel_l2(y[rows], oracle.apply_rows(oracle_mesh(P), P.x, rows)) <= TOL


def test_launches_per_apply_matches_profiler():
    """elas_launches_per_apply equals the kernels torch's profiler sees for one apply."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    from torch.profiler import profile, ProfilerActivity
    for faces, det in [(0, False), (1, False), (1, True), (0, True)]:
        P = synth.make_problem("t", 4, 3, 5, 3, 5, perturb=True, faces=faces, seed=9)
        op = Operator.from_problem(P)
        op.set_deterministic(det)
        x = torch.from_numpy(P.x).cuda()
        y = torch.empty_like(x)
        op.apply(x, y)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            op.apply(x, y)
            torch.cuda.synchronize()
        kernels = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
                   and "Memset" not in e.name and "memset" not in e.name]
        assert len(kernels) == op.launches_per_apply, (faces, det, [k.name for k in kernels])
        op.close()


def test_kernel_family_per_degree_and_mode():
    """Which kernel runs: the fine-grained FP64 kernel for p = 5..8 in the plain,
    deterministic, geometry-on-the-fly and anisotropic modes; the folded x-line kernel for p = 2..4
    and for the FP32 operator; each checked against the oracle on the same small mesh."""
    torch = torch_mod()
    import numpy as np
    from paper_2601_08374_b200.elas import Operator, VARIANT_FOLDED_OTF, VARIANT_FOLDED_F32
    from torch.profiler import profile, ProfilerActivity

    def kernel_names(op, x, y):
        op.apply(x, y)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            op.apply(x, y)
            torch.cuda.synchronize()
        return [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
                and "apply" in e.name]

    for p in range(2, 9):
        P = synth.make_problem("fam", 3, 2, 3, p, p + 2, perturb=True, lognormal_material=True, faces=1, seed=31 + p)
        x = torch.from_numpy(P.x).cuda()
        y = torch.empty_like(x)
        ref = oracle.apply(oracle_mesh(P), P.x)
        C6 = synth.random_C6(np.random.default_rng(p), (P.nz, P.ny, P.nx))
        lam, mu = P.material_arrays()
        ref_an = oracle.apply(oracle.Mesh(P.vertex_array(), P.p, P.q, lam, mu, P.dirichlet_faces, C6=C6), P.x)
        modes = [("auto", lambda: Operator.from_problem(P), None, ref)]
        if p >= 5:
            modes += [("otf", lambda: Operator.from_problem(P, variant=VARIANT_FOLDED_OTF), None, ref),
                      ("det", lambda: Operator.from_problem(P), "det", ref),
                      ("aniso", lambda: Operator.anisotropic(P, C6), None, ref_an)]
        for name, make, flag, want_y in modes:
            op = make()
            if flag == "det":
                op.set_deterministic(True)
            names = kernel_names(op, x, y)
            want = "apply_fg_kernel" if p >= 5 else "apply_eo_kernel"
            assert names and all(want in n for n in names), (p, name, names)
            assert rel_l2(y.cpu().numpy(), want_y) <= TOL, (p, name)
            op.close()
    # FP32 operator: x-line kernel at every degree
    P = synth.make_problem("fam32", 2, 2, 2, 6, 8, perturb=True, seed=5)
    x = torch.from_numpy(P.x).cuda()
    y = torch.empty_like(x)
    op = Operator.from_problem(P, variant=VARIANT_FOLDED_F32)
    names = kernel_names(op, x, y)
    assert names and all("apply_eo_kernel" in n and "float" in n for n in names), names
    op.close()


# ---------------------------------------------------------------------------------------
# general anisotropic material (Eq. 2)
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("p", range(1, 9))
def test_anisotropic_vs_oracle(p):
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = synth.make_problem("t", 3, 2, 2, p, p + 2, perturb=True, faces=1 | 32, seed=600 + p)
    C6 = synth.random_C6(np.random.default_rng(p), (P.nz, P.ny, P.nx))
    lam, mu = P.material_arrays()
    m = oracle.Mesh(P.vertex_array(), P.p, P.q, lam, mu, P.dirichlet_faces, C6=C6)
    op = Operator.anisotropic(P, C6)
    y = gpu_apply(P, op=op)
    d = torch.empty(P.num_dofs, dtype=torch.float64, device="cuda")
    op.diagonal(d)
    op.set_deterministic(True)
    y2 = gpu_apply(P, op=op)
    op.close()
    assert rel_l2(y, oracle.apply(m, P.x)) <= TOL
    assert rel_l2(y2, y) <= 1e-14
    d_ref = oracle.diagonal(m)
    assert np.abs(d.cpu().numpy() - d_ref).max() <= 1e-12 * np.abs(d_ref).max()


def test_anisotropic_isotropic_voigt_equals_isotropic_op():
    """A single isotropic Voigt matrix through elas_create_aniso == the isotropic operator."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = synth.make_problem("t", 4, 3, 5, 4, 6, perturb=True, lam=1.3, mu=0.7, faces=1, seed=61)
    op_i = Operator.from_problem(P)
    op_a = Operator.anisotropic(P, synth.isotropic_C6(1.3, 0.7))
    yi, ya = gpu_apply(P, op=op_i), gpu_apply(P, op=op_a)
    op_i.close(); op_a.close()
    assert rel_l2(ya, yi) <= 1e-13


@pytest.mark.parametrize("faces,variant", [(0, 0), (63, 0), (1 | 8 | 16, 4), (63, 3), (2 | 32, 2), (1 | 16, 8), (63, 9)])
def test_apply_add_accumulates(faces, variant):
    """elas_apply_add: y += A x with identity rows counted once on edges/corners of several faces."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    p, q = (1, 3) if variant == 3 else (6, 8) if variant == 2 else (3, 5)
    P = synth.make_problem("t", 3, 2, 4, p, q, perturb=True, lognormal_material=True, faces=faces, seed=81)
    op = Operator.from_problem(P, variant=variant)
    x = torch.from_numpy(P.x).cuda()
    y0 = torch.from_numpy(synth.splitmix_uniform(P.num_dofs, 4)).cuda()
    y = y0.clone()
    op.apply_add(x, y)
    Ax = torch.empty_like(x)
    op.apply(x, Ax)
    torch.cuda.synchronize()
    op.close()
    assert rel_l2((y - y0).cpu().numpy(), Ax.cpu().numpy()) <= 1e-14


@pytest.mark.parametrize("p", [2, 3, 4, 6])
def test_coexisting_operators_constant_tables(p):
    """The folded kernels read their 1D tables from a per-(p, q, precision) constant bank written at
    elas_create: operators of both quadrature orders and both precisions,
    created before any of them applies, each still match the oracle."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator, VARIANT_FOLDED, VARIANT_FOLDED_F32, VARIANT_FOLDED_OTF
    probs = [synth.make_problem(f"ct_p{p}_q{p + dq}", 3, 2, 2, p, p + dq, perturb=True,
                                lognormal_material=True, faces=1 | 16, seed=40 + dq) for dq in (1, 2)]
    ops = [(P, v, Operator.from_problem(P, variant=v)) for P in probs
           for v in (VARIANT_FOLDED, VARIANT_FOLDED_F32, VARIANT_FOLDED_OTF)]
    for P, v, op in reversed(ops):
        y = gpu_apply(P, op=op)
        tol = TOL_F32 if v == VARIANT_FOLDED_F32 else TOL
        assert rel_l2(y, oracle.apply(oracle_mesh(P), P.x)) <= tol, (P.name, v)
    for _, _, op in ops:
        op.close()


@pytest.mark.parametrize("p,dims,faces", [(1, (64, 64, 64), 63), (2, (40, 41, 161), 1 | 16 | 32), (3, (48, 40, 150), 2 | 8)])
def test_pipelined_zeroing_chunk_planes(p, dims, faces):
    """Large operators (>= 2^18 elements, the size where elas_apply may pipeline the zeroing of
    y over 8 z-chunks, ELAS_INIT_CHUNKS): rows on the eighth-planes (chunk boundaries), on the
    Dirichlet faces and at random match the oracle; identity rows are exact; applying into a y
    that already holds a result overwrites all of it."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    nx, ny, nz = dims
    P = synth.make_problem("pz", nx, ny, nz, p, p + 1, perturb=True, lognormal_material=True, faces=faces, seed=77)
    assert P.num_elements >= 1 << 18
    Nx, Ny, Nz = P.node_dims
    N = Nx * Ny * Nz
    chunk_planes = [((k * nz) // 8) * p for k in range(1, 8)]
    extra = np.concatenate([plane_rows(P, K + d, 24, K + d) for K in chunk_planes for d in (-1, 0, 1)]
                           + [np.arange(0, N, Nx)[:40]])
    rows = sample_rows(P, 256, 3, extra=extra)
    op = Operator.from_problem(P)
    xd = torch.from_numpy(P.x).cuda()
    yd = torch.full_like(xd, 1e300)
    op.apply(xd, yd)
    op.apply(xd, yd)          # y already holds a result: the chunked zeroing must clear all of it
    torch.cuda.synchronize()
    y = yd.cpu().numpy()
    op.close()
    m = oracle_mesh(P)
    assert rel_l2(y[rows], oracle.apply_rows(m, P.x, rows)) <= TOL
    Z = oracle.constrained_mask(m)
    assert np.array_equal(y[Z], P.x[Z])
    assert np.all(np.abs(y) < 1e100)


@pytest.mark.parametrize("p,variant", [(1, 6), (2, 6), (8, 6), (2, 5), (8, 5)])
def test_config4_full_size_otf_and_f32(p, variant):
    """Full-size config 4 for the geometry-on-the-fly (6; p = 1 runs the thread-per-element
    kernel) and mixed-precision (5) operators: sampled rows vs the oracle at each contract."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = synth.make_config(4, p)
    op = Operator.from_problem(P, variant=variant)
    assert op.variant == variant
    x = torch.from_numpy(P.x).cuda()
    y = torch.empty_like(x)
    op.apply(x, y)
    torch.cuda.synchronize()
    op.close()
    yh = y.cpu().numpy()
    rows = sample_rows(P, 160, 70 + p, extra=plane_rows(P, P.p * 3, 16, p))
    y_ref = oracle.apply_rows(oracle_mesh(P), P.x, rows)
    assert rel_l2(yh[rows], y_ref) <= (TOL_F32 if variant == 5 else TOL)


@pytest.mark.parametrize("p", [2, 6])
def test_anisotropic_config4_sampled(p):
    """Full-size config 4 with a random SPD Voigt matrix per element (the bench's anisotropic
    row): sampled rows vs the oracle."""
    torch = torch_mod()
    from paper_2601_08374_b200.elas import Operator
    P = synth.make_config(4, p)
    C6 = synth.random_C6(np.random.default_rng(90 + p), (P.nz, P.ny, P.nx))
    lam, mu = P.material_arrays()
    m = oracle.Mesh(P.vertex_array(), P.p, P.q, lam, mu, P.dirichlet_faces, C6=C6)
    op = Operator.anisotropic(P, C6)
    x = torch.from_numpy(P.x).cuda()
    y = torch.empty_like(x)
    op.apply(x, y)
    torch.cuda.synchronize()
    op.close()
    rows = sample_rows(P, 160, 80 + p, extra=plane_rows(P, P.p * 3, 16, p))
    assert rel_l2(y.cpu().numpy()[rows], oracle.apply_rows(m, P.x, rows)) <= TOL
