"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no basis, quadrature, geometry factors or
operator).  It only draws the inputs the configurations of BASELINE.json describe, in the
order fixed by DESIGN.md reading R11:

  rng = numpy.random.default_rng(seed)          (PCG64)
  (1) vertex perturbation, shape (nz+1, ny+1, nx+1, 3), uniform(-0.1 h, 0.1 h);
      the boundary-normal component of boundary vertices is then zeroed (reading R7)
  (2) lambda_e, shape (nz, ny, nx), lognormal(0, 0.5)          (reading R12)
  (3) mu_e, same
  (4) x, shape (3, Nz, Ny, Nx), uniform(-1, 1)
Items absent from a configuration are skipped (no draw).

The paper's own benchmark problem (geometry, load, Lame values) is unstated;
these configurations stand in for it at the paper's sizes.
"""

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

FACE_XMIN = 1


@dataclass
class Problem:
    name: str
    nx: int
    ny: int
    nz: int
    p: int
    q: int
    lx: float
    ly: float
    lz: float
    vertices: Optional[np.ndarray]     # None => uniform (affine) grid
    lam: np.ndarray                    # shape () for constant or (nz, ny, nx)
    mu: np.ndarray
    x: Optional[np.ndarray]            # (3 * Nx * Ny * Nz,) component-blocked, or None (lazy)
    dirichlet_faces: int = 0
    seed: int = 0
    x_rng_state: dict = field(default=None, repr=False)  # PCG64 state right before the x draw

    @property
    def node_dims(self):
        return self.nx * self.p + 1, self.ny * self.p + 1, self.nz * self.p + 1

    @property
    def num_dofs(self):
        Nx, Ny, Nz = self.node_dims
        return 3 * Nx * Ny * Nz

    @property
    def num_elements(self):
        return self.nx * self.ny * self.nz

    @property
    def per_element_material(self):
        return np.ndim(self.lam) == 3

    def vertex_array(self):
        """Vertex coordinates (nz+1, ny+1, nx+1, 3); builds the uniform grid when affine."""
        if self.vertices is not None:
            return self.vertices
        return uniform_vertices(self.nx, self.ny, self.nz, self.lx, self.ly, self.lz)

    def material_arrays(self):
        shape = (self.nz, self.ny, self.nx)
        return (np.broadcast_to(np.asarray(self.lam, dtype=np.float64), shape),
                np.broadcast_to(np.asarray(self.mu, dtype=np.float64), shape))

    def x_slab(self, K0, K1):
        """Rows K in [K0, K1] (inclusive) of x, component-blocked, drawn by advancing PCG64.

        Equal to x.reshape(3, Nz, Ny, Nx)[:, K0:K1+1].reshape(-1) without drawing all of x.
        """
        Nx, Ny, Nz = self.node_dims
        plane = Nx * Ny
        out = np.empty((3, K1 - K0 + 1, Ny, Nx))
        for c in range(3):
            bg = np.random.PCG64()
            bg.state = self.x_rng_state
            bg.advance(c * Nz * plane + K0 * plane)
            out[c] = np.random.Generator(bg).uniform(-1.0, 1.0, size=(K1 - K0 + 1, Ny, Nx))
        return out.reshape(-1)


def uniform_vertices(nx, ny, nz, lx, ly, lz):
    X = np.linspace(0.0, lx, nx + 1)
    Y = np.linspace(0.0, ly, ny + 1)
    Zc = np.linspace(0.0, lz, nz + 1)
    V = np.empty((nz + 1, ny + 1, nx + 1, 3))
    V[..., 0] = X[None, None, :]
    V[..., 1] = Y[None, :, None]
    V[..., 2] = Zc[:, None, None]
    return V


def perturbed_vertices(rng, nx, ny, nz, lx, ly, lz, h):
    """Uniform grid plus U[-0.1h, 0.1h] per coordinate; boundary-normal components zeroed."""
    V = uniform_vertices(nx, ny, nz, lx, ly, lz)
    d = rng.uniform(-0.1 * h, 0.1 * h, size=V.shape)
    d[:, :, 0, 0] = 0.0
    d[:, :, -1, 0] = 0.0
    d[:, 0, :, 1] = 0.0
    d[:, -1, :, 1] = 0.0
    d[0, :, :, 2] = 0.0
    d[-1, :, :, 2] = 0.0
    return V + d


def make_problem(name, nx, ny, nz, p, q, *, lengths=(1.0, 1.0, 1.0), perturb=False,
                 lam=1.0, mu=1.0, lognormal_material=False, faces=0, seed=0, draw_x=True):
    lx, ly, lz = lengths
    rng = np.random.default_rng(seed)
    V = None
    if perturb:
        h = min(lx / nx, ly / ny, lz / nz)
        V = perturbed_vertices(rng, nx, ny, nz, lx, ly, lz, h)
    if lognormal_material:
        lam_a = rng.lognormal(0.0, 0.5, size=(nz, ny, nx))
        mu_a = rng.lognormal(0.0, 0.5, size=(nz, ny, nx))
    else:
        lam_a = np.asarray(float(lam))
        mu_a = np.asarray(float(mu))
    state = rng.bit_generator.state
    Nx, Ny, Nz = nx * p + 1, ny * p + 1, nz * p + 1
    x = rng.uniform(-1.0, 1.0, size=(3, Nz, Ny, Nx)).reshape(-1) if draw_x else None
    return Problem(name, nx, ny, nz, p, q, lx, ly, lz, V, lam_a, mu_a, x, faces, seed, state)


def config4_elements(p):
    """Config 4: hex count per axis = round((5e7/3)^(1/3) / p)  (reading R13)."""
    return int(round((5e7 / 3.0) ** (1.0 / 3.0) / p))


def make_config(cfg, p=None, draw_x=True):
    """The five configurations of BASELINE.json (configs[cfg-1])."""
    if cfg == 1:
        return make_problem("cfg1", 2, 2, 2, 2, 4, lam=1.0, mu=1.0, seed=0, draw_x=draw_x)
    if cfg == 2:
        return make_problem("cfg2", 16, 16, 16, 4, 6, perturb=True, lam=1.5, mu=1.0, seed=1,
                            draw_x=draw_x)
    if cfg == 3:
        return make_problem("cfg3", 24, 24, 24, 6, 8, perturb=True, lognormal_material=True,
                            faces=FACE_XMIN, seed=2, draw_x=draw_x)
    if cfg == 4:
        if p is None:
            raise ValueError("config 4 needs p")
        m = config4_elements(p)
        return make_problem(f"cfg4_p{p}", m, m, m, p, p + 2, lam=1.0, mu=0.5, seed=3,
                            draw_x=draw_x)
    if cfg == 5:
        return make_problem("cfg5", 64, 64, 256, 6, 8, lengths=(1.0, 1.0, 4.0), perturb=True,
                            lognormal_material=True, seed=4, draw_x=draw_x)
    raise ValueError(f"unknown config {cfg}")


def splitmix_uniform(n, seed):
    """Counter-based draw in [-1, 1): u_i = 2 * (splitmix64(seed, i) >> 11) * 2^-53 - 1.

    splitmix64(seed, i): z = seed + (i + 1) * 0x9E3779B97F4A7C15 (mod 2^64);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9; z = (z ^ (z >> 27)) * 0x94D049BB133111EB;
    z ^= z >> 31.  The power-iteration start vector (reading R19); libelas implements
    the same counter-based generator for its default start vector.
    """
    with np.errstate(over="ignore"):
        i = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return 2.0 * (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) - 1.0


def isotropic_C6(lam, mu):
    """The 6x6 Voigt matrix of Hooke's law (Eq. 3) -- an input-construction helper (no operator)."""
    C = np.zeros((6, 6))
    C[:3, :3] = lam
    C[[0, 1, 2], [0, 1, 2]] = lam + 2 * mu
    C[[3, 4, 5], [3, 4, 5]] = mu
    return C


def random_C6(rng, shape, scale=1.0):
    """Seeded symmetric positive-definite 6x6 Voigt matrices (general anisotropic materials, Eq. 2):
    C = L L^T + 0.5 I with L ~ N(0, 0.3^2) entries, times `scale`; shape (..., 6, 6)."""
    L = rng.normal(0.0, 0.3, size=tuple(shape) + (6, 6))
    return scale * (L @ np.swapaxes(L, -1, -2) + 0.5 * np.eye(6))
