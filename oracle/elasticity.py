"""Oracle: element stiffness matrices by naive quadrature, applied element by element.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py for who may import this).

Definitions followed, step by step:
* Operator: A_ij = a(phi_i, phi_j), PAPER.md:158-162 (Eq. 5), with
  a(u, v) = int sigma(u) : grad v  (Eq. 4, the "alternative form") and
  sigma(u) = lambda (div u) I + 2 mu eps(u)  (Eq. 3).
  Substituting u = phi_J e_j and v = phi_I e_i gives the entry
      K[(i,I),(j,J)] = int lambda d_i phi_I d_j phi_J + mu d_j phi_I d_i phi_J
                              + mu delta_ij grad phi_I . grad phi_J .
* Basis: Phi_ijk(xi, eta, zeta) = phi_i(xi) phi_j(eta) phi_k(zeta), PAPER.md:192-194 (Eq. 6),
  Lagrange on GLL nodes (reading R2).
* Geometry: trilinear hexahedra ("structured mesh of trilinear hexahedral elements",
  PAPER.md:391); J_mk = d x_m / d xi_k; physical gradient grad_x phi = grad_xi phi . J^{-1}.
* Quadrature: q-point Gauss-Legendre per direction on [0,1]^3, weight w_a w_b w_c det J
  (Alg. 1 "w_p det(J)").
* Element matrices assembled/applied through the element restriction G and its transpose
  (operator chain A = P^T G^T B^T D B G P): "explicitly calculating each
  local matrix".
* Dirichlet faces: y = Z A Z x + (I - Z) x (rows and columns zeroed, unit diagonal), the
  reading R9 in DESIGN.md.

Numbering (reading R6): global node (I,J,K) -> I + Nx (J + Ny K), Nx = nx p + 1; element
(ex,ey,ez) -> ex + nx (ey + ny ez); element-local node (i,j,k) -> i + n (j + n k), n = p+1;
vectors are component-blocked: dof = c N + node (local: c n^3 + l).
"""

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .rules import gauss_legendre, gll_nodes, lagrange_derivatives, lagrange_values

FACE_XMIN, FACE_XMAX, FACE_YMIN, FACE_YMAX, FACE_ZMIN, FACE_ZMAX = 1, 2, 4, 8, 16, 32


@dataclass
class Mesh:
    """Structured hex mesh with vertex coordinates V[k, j, i, 0:3] (x fastest)."""

    vertices: np.ndarray          # (nz+1, ny+1, nx+1, 3)
    p: int
    q: int
    lam: np.ndarray               # (nz, ny, nx) per-element lambda
    mu: np.ndarray                # (nz, ny, nx) per-element mu
    dirichlet_faces: int = 0
    C6: Optional[np.ndarray] = None   # anisotropic (Eq. 2): (nz, ny, nx, 6, 6) Voigt matrices; replaces lam, mu

    def __post_init__(self):
        self.vertices = np.ascontiguousarray(self.vertices, dtype=np.float64)
        nz1, ny1, nx1, three = self.vertices.shape
        assert three == 3
        self.nx, self.ny, self.nz = nx1 - 1, ny1 - 1, nz1 - 1
        shape = (self.nz, self.ny, self.nx)
        self.lam = np.broadcast_to(np.asarray(self.lam, dtype=np.float64), shape)
        self.mu = np.broadcast_to(np.asarray(self.mu, dtype=np.float64), shape)
        if self.C6 is not None:
            self.C6 = np.broadcast_to(np.asarray(self.C6, dtype=np.float64), shape + (6, 6))

    @property
    def n(self):
        return self.p + 1

    @property
    def node_dims(self):
        p = self.p
        return self.nx * p + 1, self.ny * p + 1, self.nz * p + 1

    @property
    def num_nodes(self):
        Nx, Ny, Nz = self.node_dims
        return Nx * Ny * Nz

    @property
    def num_dofs(self):
        return 3 * self.num_nodes


# ----------------------------------------------------------------------------------------
# Reference tables (Eq. 6): d/dxi_k of every scalar basis function at every quadrature point
# ----------------------------------------------------------------------------------------

def reference_tables(p, q):
    """Return (Gref, w3): Gref[k] is (n^3, q^3) with d phi_l / d xi_k at qp, w3 the q^3 weights.

    Local node l = i + n (j + n k); quadrature point index a1 + q (a2 + q a3).
    """
    nodes = gll_nodes(p)
    g, w = gauss_legendre(q)
    B = lagrange_values(nodes, g)       # B[a, i] = l_i(g_a)
    D = lagrange_derivatives(nodes, g)  # D[a, i] = l_i'(g_a)
    n = p + 1
    # Eq. 6 outer products; array axes (k, j, i, a3, a2, a1)
    G0 = np.einsum("ck,bj,ai->kjicba", B, B, D).reshape(n ** 3, q ** 3)
    G1 = np.einsum("ck,bj,ai->kjicba", B, D, B).reshape(n ** 3, q ** 3)
    G2 = np.einsum("ck,bj,ai->kjicba", D, B, B).reshape(n ** 3, q ** 3)
    w3 = np.einsum("c,b,a->cba", w, w, w).reshape(q ** 3)
    return np.stack([G0, G1, G2]), w3, g


def element_vertices(mesh, ex, ey, ez):
    """X[c, b, a, :] = coordinates of vertex (ex+a, ey+b, ez+c)."""
    return mesh.vertices[ez:ez + 2, ey:ey + 2, ex:ex + 2, :]


def element_geometry(X, g, w3):
    """Trilinear Jacobian at the q^3 Gauss points: returns (J (q^3,3,3), detJ, W = w detJ)."""
    q = g.size
    hat = [1.0 - g, g]
    dhat = [-np.ones_like(g), np.ones_like(g)]
    J = np.zeros((q, q, q, 3, 3))        # axes (a3, a2, a1, m, k)
    for c in range(2):
        for b in range(2):
            for a in range(2):
                Xv = X[c, b, a]
                d0 = np.einsum("c,b,a->cba", hat[c], hat[b], dhat[a])
                d1 = np.einsum("c,b,a->cba", hat[c], dhat[b], hat[a])
                d2 = np.einsum("c,b,a->cba", dhat[c], hat[b], hat[a])
                for m in range(3):
                    J[..., m, 0] += Xv[m] * d0
                    J[..., m, 1] += Xv[m] * d1
                    J[..., m, 2] += Xv[m] * d2
    J = J.reshape(q ** 3, 3, 3)
    detJ = np.linalg.det(J)
    if np.any(detJ <= 0.0):
        raise ValueError("non-positive Jacobian determinant")
    return J, detJ, w3 * detJ


def element_stiffness(X, lam, mu, tables, rows=None):
    """Element stiffness K_e (3n^3 x 3n^3, component-blocked) or only the given local rows.

    rows: None (all) or an int array of local dofs r = c n^3 + l.
    K[(i,I),(j,J)] = sum_qp W [lam d_i phi_I d_j phi_J + mu d_j phi_I d_i phi_J
                               + mu delta_ij grad phi_I . grad phi_J]      (Eqs. 3-5)
    """
    Gref, w3, g = tables
    nn = Gref.shape[1]
    J, detJ, W = element_geometry(X, g, w3)
    A = np.linalg.inv(J)                                   # A = J^{-1}, (q^3, 3, 3)
    # physical gradients Phi[m][l, qp] = sum_k Gref[k][l, qp] A[qp, k, m]
    Phi = np.einsum("klq,qkm->mlq", Gref, A, optimize=True)
    if rows is None:
        rows = np.arange(3 * nn)
    rows = np.asarray(rows)
    comp, node = rows // nn, rows % nn
    # M[k][l][r, J] = sum_qp W Phi_k[node_r, qp] Phi_l[J, qp]
    PW = Phi[:, node, :] * W                               # (3, R, q^3)
    M = np.einsum("krq,lJq->klrJ", PW, Phi, optimize=True)  # (3, 3, R, n^3)
    trace = M[0, 0] + M[1, 1] + M[2, 2]                    # (R, n^3)
    R = rows.size
    r = np.arange(R)
    # row r = (i, I) with i = comp[r]; block j: lam M[i, j, r] + mu M[j, i, r] (+ mu tr if i == j)
    K = lam * M[comp, :, r, :] + mu * M[:, comp, r, :].transpose(1, 0, 2)   # (R, 3, n^3)
    K[r, comp, :] += mu * trace
    return K.reshape(R, 3 * nn)


VOIGT = np.array([[0, 5, 4], [5, 1, 3], [4, 3, 2]])   # (i, j) -> Voigt index [11,22,33,23,13,12]


def element_stiffness_aniso(X, C6, tables, rows=None):
    """Element stiffness for a general anisotropic material (Eq. 2):
    sigma_voigt = C eps_voigt with eps_voigt = [e11, e22, e33, 2e23, 2e13, 2e12],
    i.e. C_ijkl = C6[v(i,j)][v(k,l)], and
        K[(i,I),(j,J)] = sum_qp W sum_{k,l} d_k phi_I C_ikjl d_l phi_J .
    """
    Gref, w3, g = tables
    nn = Gref.shape[1]
    J, detJ, W = element_geometry(X, g, w3)
    A = np.linalg.inv(J)
    Phi = np.einsum("klq,qkm->mlq", Gref, A, optimize=True)        # Phi[m][l, qp] = d_m phi_l
    C4 = C6[VOIGT[:, :, None, None], VOIGT[None, None, :, :]]      # C4[i, k, j, l]
    if rows is None:
        rows = np.arange(3 * nn)
    rows = np.asarray(rows)
    comp, node = rows // nn, rows % nn
    PW = Phi[:, node, :] * W                                       # (3, R, q)
    # K[r, j, J] = sum_{k,l} C4[i_r, k, j, l] sum_q PW[k, r, q] Phi[l, J, q]
    M = np.einsum("krq,lJq->klrJ", PW, Phi, optimize=True)         # (3, 3, R, n^3)
    K = np.einsum("rkjl,klrJ->rjJ", C4[comp], M, optimize=True)    # (R, 3, n^3)
    return K.reshape(rows.size, 3 * nn)


def _stiffness(mesh, ex, ey, ez, tables, rows=None):
    X = element_vertices(mesh, ex, ey, ez)
    if mesh.C6 is not None:
        return element_stiffness_aniso(X, mesh.C6[ez, ey, ex], tables, rows)
    return element_stiffness(X, mesh.lam[ez, ey, ex], mesh.mu[ez, ey, ex], tables, rows)


# ----------------------------------------------------------------------------------------
# Element restriction G (gather) and its transpose (scatter), Dirichlet mask Z
# ----------------------------------------------------------------------------------------

def element_nodes(mesh, ex, ey, ez):
    """Global node ids of the n^3 local nodes (local order i + n(j + n k))."""
    p, n = mesh.p, mesh.n
    Nx, Ny, _ = mesh.node_dims
    k, j, i = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    I = ex * p + i
    Jg = ey * p + j
    Kg = ez * p + k
    return (I + Nx * (Jg + Ny * Kg)).reshape(-1)


def constrained_mask(mesh):
    """Boolean mask over the 3N dofs: True where a Dirichlet face constrains the dof."""
    Nx, Ny, Nz = mesh.node_dims
    K, J, I = np.meshgrid(np.arange(Nz), np.arange(Ny), np.arange(Nx), indexing="ij")
    f = mesh.dirichlet_faces
    m = np.zeros((Nz, Ny, Nx), dtype=bool)
    if f & FACE_XMIN: m |= I == 0
    if f & FACE_XMAX: m |= I == Nx - 1
    if f & FACE_YMIN: m |= J == 0
    if f & FACE_YMAX: m |= J == Ny - 1
    if f & FACE_ZMIN: m |= K == 0
    if f & FACE_ZMAX: m |= K == Nz - 1
    return np.tile(m.reshape(-1), 3)


def _elements(mesh):
    for ez in range(mesh.nz):
        for ey in range(mesh.ny):
            for ex in range(mesh.nx):
                yield ex, ey, ez


def apply(mesh, x):
    """y = Z A Z x + (I - Z) x, element by element (full mode)."""
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    assert x.size == mesh.num_dofs
    Z = constrained_mask(mesh)
    y = apply_elements(mesh, np.where(Z, 0.0, x), _elements(mesh))
    y[Z] = x[Z]
    return y


def apply_elements(mesh, xz, elements):
    """sum_e G_e^T K_e G_e xz over the given elements (x already masked); the loop of apply."""
    N = mesh.num_nodes
    tables = reference_tables(mesh.p, mesh.q)
    y = np.zeros(3 * N)
    for ex, ey, ez in elements:
        nodes = element_nodes(mesh, ex, ey, ez)
        dofs = np.concatenate([c * N + nodes for c in range(3)])
        K = _stiffness(mesh, ex, ey, ez, tables)
        np.add.at(y, dofs, K @ xz[dofs])
    return y


def apply_rows(mesh, x, dofs):
    """Sampled-row mode: y[dofs] of the same operator, touching only elements that hold them."""
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    dofs = np.asarray(dofs, dtype=np.int64).reshape(-1)
    N = mesh.num_nodes
    Nx, Ny, _ = mesh.node_dims
    p, n = mesh.p, mesh.n
    Z = constrained_mask(mesh)
    xz = np.where(Z, 0.0, x)
    tables = reference_tables(p, q=mesh.q)
    # group (row position, local row) by element
    work = {}
    for pos, dof in enumerate(dofs):
        if Z[dof]:
            continue
        c, node = divmod(int(dof), N)
        I = node % Nx
        Jg = (node // Nx) % Ny
        Kg = node // (Nx * Ny)

        def owners(G, ne):
            return [e for e in (G // p - 1, G // p) if 0 <= e < ne and e * p <= G <= (e + 1) * p]

        for ez in owners(Kg, mesh.nz):
            for ey in owners(Jg, mesh.ny):
                for ex in owners(I, mesh.nx):
                    l = (I - ex * p) + n * ((Jg - ey * p) + n * (Kg - ez * p))
                    work.setdefault((ex, ey, ez), []).append((pos, c * n ** 3 + l))
    y = np.where(Z[dofs], x[dofs], 0.0)
    for (ex, ey, ez), lst in work.items():
        nodes = element_nodes(mesh, ex, ey, ez)
        edofs = np.concatenate([c * N + nodes for c in range(3)])
        pos = np.array([a for a, _ in lst])
        lrows = np.array([b for _, b in lst])
        K = _stiffness(mesh, ex, ey, ez, tables, rows=lrows)
        np.add.at(y, pos, K @ xz[edofs])
    return y


def assemble_dense(mesh):
    """Dense global A (with Dirichlet rows/cols replaced by identity). Tiny meshes only."""
    N = mesh.num_nodes
    A = np.zeros((3 * N, 3 * N))
    tables = reference_tables(mesh.p, mesh.q)
    for ex, ey, ez in _elements(mesh):
        nodes = element_nodes(mesh, ex, ey, ez)
        dofs = np.concatenate([c * N + nodes for c in range(3)])
        K = _stiffness(mesh, ex, ey, ez, tables)
        A[np.ix_(dofs, dofs)] += K
    Z = constrained_mask(mesh)
    A[Z, :] = 0.0
    A[:, Z] = 0.0
    A[Z, Z] = 1.0
    return A


def node_coordinates(mesh):
    """Physical coordinates (N, 3) of every global node (GLL node mapped trilinearly)."""
    p = mesh.p
    xi = gll_nodes(p)
    Nx, Ny, Nz = mesh.node_dims

    def split(G, ne):
        e = np.minimum(G // p, ne - 1)
        return e, xi[G - e * p]

    K, J, I = np.meshgrid(np.arange(Nz), np.arange(Ny), np.arange(Nx), indexing="ij")
    ex, s = split(I.reshape(-1), mesh.nx)
    ey, t = split(J.reshape(-1), mesh.ny)
    ez, u = split(K.reshape(-1), mesh.nz)
    V = mesh.vertices
    out = np.zeros((ex.size, 3))
    for c in range(2):
        for b in range(2):
            for a in range(2):
                wgt = (s if a else 1 - s) * (t if b else 1 - t) * (u if c else 1 - u)
                out += wgt[:, None] * V[ez + c, ey + b, ex + a]
    return out
