"""Thin ctypes binding of libelas.so (include/elas.h): argument marshalling only.

Every step of the operator runs in the library's CUDA kernels.  There is no CPU fallback:
if the in-tree library is missing, ``load()`` raises (build it with
``python -m paper_2601_08374_b200.build`` or ``__graft_entry__.build()``).

Functions mirror the C names (elas_create, elas_apply, ...); ``Operator`` is a small
convenience wrapper that owns the handle.  Device arrays are passed as torch CUDA tensors
(or raw integer device pointers); host arrays as numpy float64 arrays.
"""

import ctypes
import weakref
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", os.environ.get("ELAS_LIBNAME", "libelas.so"))

VARIANT_AUTO, VARIANT_SIMT, VARIANT_TENSOR, VARIANT_THREAD, VARIANT_FOLDED, VARIANT_FOLDED_F32, VARIANT_FOLDED_OTF = (
    0, 1, 2, 3, 4, 5, 6)
# the paper's ablation stages (Table 4) as unfused pipelines, for measurement (include/elas.h)
VARIANT_ABL_PA, VARIANT_ABL_SF, VARIANT_ABL_VOIGT = 7, 8, 9
ELAS_OK, ELAS_EINVAL, ELAS_EGEOM, ELAS_ENOMEM, ELAS_ECUDA, ELAS_ENCCL = 0, -1, -2, -3, -4, -5
FACE_XMIN, FACE_XMAX, FACE_YMIN, FACE_YMAX, FACE_ZMIN, FACE_ZMAX = 1, 2, 4, 8, 16, 32

EXPORTED = ["elas_create", "elas_apply", "elas_apply_host", "elas_interface_add", "elas_destroy",
            "elas_local_dofs", "elas_local_zrange", "elas_set_stream", "elas_launches_per_apply",
            "elas_last_error", "elas_slab_range", "elas_tables", "elas_nccl_unique_id", "elas_version",
            "elas_profile", "elas_profile_read", "elas_create_ex", "elas_variant",
            "elas_diagonal", "elas_cheb_create", "elas_cheb_lambda_max", "elas_cheb_apply",
            "elas_cheb_destroy", "elas_pcg", "elas_gmg_create", "elas_gmg_level_op", "elas_gmg_levels",
            "elas_gmg_set_stream", "elas_gmg_apply", "elas_pcg_gmg", "elas_gmg_destroy", "elas_gmg_transfer",
            "elas_set_deterministic", "elas_dot", "elas_create_aniso", "elas_apply_add",
            "elas_set_peer_exchange", "elas_debug_checks", "elas_debug_build"]
PC_NONE, PC_JACOBI, PC_CHEBYSHEV = 0, 1, 2


class ElasError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"elas error {code}: {msg}")
        self.code = code


class elas_solve_report(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("converged", ctypes.c_int), ("rel_residual", ctypes.c_double)]


class elas_mesh(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("vertices", ctypes.POINTER(ctypes.c_double)),
                ("lx", ctypes.c_double), ("ly", ctypes.c_double), ("lz", ctypes.c_double),
                ("dirichlet_faces", ctypes.c_uint32), ("material_per_element", ctypes.c_int32),
                ("nccl_id", ctypes.c_void_p), ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32)]


_lib = None


def load(path=None):
    """Load the in-tree libelas.so (raises if it is missing: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(f"libelas.so not built at {path}; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    P, D, I32, I64 = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int32, ctypes.c_int64
    lib.elas_create.restype = P
    lib.elas_create.argtypes = [ctypes.POINTER(elas_mesh), ctypes.c_int, ctypes.c_int, D, D]
    lib.elas_create_ex.restype = P
    lib.elas_create_ex.argtypes = [ctypes.POINTER(elas_mesh), ctypes.c_int, ctypes.c_int, D, D, ctypes.c_int]
    lib.elas_variant.restype = ctypes.c_int
    lib.elas_variant.argtypes = [P]
    lib.elas_apply.restype = ctypes.c_int
    lib.elas_apply.argtypes = [P, P, P]
    lib.elas_apply_host.restype = ctypes.c_int
    lib.elas_apply_host.argtypes = [P, P, P]
    lib.elas_interface_add.restype = ctypes.c_int
    lib.elas_interface_add.argtypes = [P, P, P, P]
    lib.elas_destroy.restype = None
    lib.elas_destroy.argtypes = [P]
    lib.elas_local_dofs.restype = I64
    lib.elas_local_dofs.argtypes = [P]
    lib.elas_local_zrange.restype = ctypes.c_int
    lib.elas_local_zrange.argtypes = [P, ctypes.POINTER(I32), ctypes.POINTER(I32)]
    lib.elas_set_stream.restype = ctypes.c_int
    lib.elas_set_stream.argtypes = [P, P]
    lib.elas_launches_per_apply.restype = ctypes.c_int
    lib.elas_launches_per_apply.argtypes = [P]
    lib.elas_last_error.restype = ctypes.c_char_p
    lib.elas_last_error.argtypes = []
    lib.elas_slab_range.restype = ctypes.c_int
    lib.elas_slab_range.argtypes = [I32, I32, I32, ctypes.POINTER(I32), ctypes.POINTER(I32)]
    lib.elas_tables.restype = ctypes.c_int
    lib.elas_tables.argtypes = [ctypes.c_int, ctypes.c_int, D, D, D, D, D]
    lib.elas_version.restype = ctypes.c_int
    lib.elas_version.argtypes = []
    lib.elas_nccl_unique_id.restype = ctypes.c_int
    lib.elas_nccl_unique_id.argtypes = [P]
    lib.elas_profile.restype = ctypes.c_int
    lib.elas_profile.argtypes = [P, ctypes.c_int]
    lib.elas_profile_read.restype = ctypes.c_int
    lib.elas_profile_read.argtypes = [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I64)]
    lib.elas_diagonal.restype = ctypes.c_int
    lib.elas_diagonal.argtypes = [P, P]
    lib.elas_cheb_create.restype = P
    lib.elas_cheb_create.argtypes = [P, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int, P,
                                     ctypes.c_ulonglong]
    lib.elas_cheb_lambda_max.restype = ctypes.c_double
    lib.elas_cheb_lambda_max.argtypes = [P]
    lib.elas_cheb_apply.restype = ctypes.c_int
    lib.elas_cheb_apply.argtypes = [P, P, P]
    lib.elas_cheb_destroy.restype = None
    lib.elas_cheb_destroy.argtypes = [P]
    lib.elas_pcg.restype = ctypes.c_int
    lib.elas_pcg.argtypes = [P, ctypes.c_int, P, P, P, ctypes.c_double, ctypes.c_int,
                             ctypes.POINTER(elas_solve_report), D]
    lib.elas_gmg_create.restype = P
    lib.elas_gmg_create.argtypes = [ctypes.POINTER(elas_mesh), ctypes.c_int, ctypes.c_int, D, D, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_ulonglong,
                                    ctypes.c_double, ctypes.c_int, ctypes.c_int]
    lib.elas_gmg_level_op.restype = P
    lib.elas_gmg_level_op.argtypes = [P, ctypes.c_int]
    lib.elas_gmg_levels.restype = ctypes.c_int
    lib.elas_gmg_levels.argtypes = [P]
    lib.elas_gmg_set_stream.restype = ctypes.c_int
    lib.elas_gmg_set_stream.argtypes = [P, P]
    lib.elas_gmg_apply.restype = ctypes.c_int
    lib.elas_gmg_apply.argtypes = [P, P, P]
    lib.elas_pcg_gmg.restype = ctypes.c_int
    lib.elas_pcg_gmg.argtypes = [P, P, P, P, ctypes.c_double, ctypes.c_int, ctypes.POINTER(elas_solve_report), D]
    lib.elas_create_aniso.restype = P
    lib.elas_create_aniso.argtypes = [ctypes.POINTER(elas_mesh), ctypes.c_int, ctypes.c_int, D]
    lib.elas_apply_add.restype = ctypes.c_int
    lib.elas_apply_add.argtypes = [P, P, P]
    lib.elas_dot.restype = ctypes.c_int
    lib.elas_dot.argtypes = [P, P, P, D]
    lib.elas_set_deterministic.restype = ctypes.c_int
    lib.elas_set_deterministic.argtypes = [P, ctypes.c_int]
    lib.elas_set_peer_exchange.restype = ctypes.c_int
    lib.elas_set_peer_exchange.argtypes = [P, ctypes.c_int]
    lib.elas_debug_checks.restype = ctypes.c_int
    lib.elas_debug_checks.argtypes = [ctypes.POINTER(ctypes.c_int), ctypes.c_int]
    lib.elas_debug_build.restype = ctypes.c_int
    lib.elas_debug_build.argtypes = []
    lib.elas_gmg_transfer.restype = ctypes.c_int
    lib.elas_gmg_transfer.argtypes = [P, ctypes.c_int, ctypes.c_int, P, P]
    lib.elas_gmg_destroy.restype = None
    lib.elas_gmg_destroy.argtypes = [P]
    _lib = lib
    return lib


def _ptr(a):
    """Device pointer of a torch tensor (or an int pointer)."""
    if a is None:
        return None
    if isinstance(a, int):
        return a
    return a.data_ptr()


def _dptr(arr):
    return arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _check(rc, what):
    if rc != ELAS_OK:
        raise ElasError(rc, f"{what}: {elas_last_error()}")


# ------------------------------------------------------------------ C-named functions

def elas_last_error():
    return load().elas_last_error().decode()


def elas_version():
    return load().elas_version()


def elas_nccl_unique_id():
    """A fresh 128-byte ncclUniqueId (bytes) for elas_create(..., nccl_id=...)."""
    buf = ctypes.create_string_buffer(128)
    _check(load().elas_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)), "elas_nccl_unique_id")
    return buf.raw


def elas_slab_range(nz, rank, nranks):
    b, e = ctypes.c_int32(), ctypes.c_int32()
    _check(load().elas_slab_range(nz, rank, nranks, ctypes.byref(b), ctypes.byref(e)), "elas_slab_range")
    return b.value, e.value


def elas_tables(p, q):
    """(nodes[p+1], points[q], weights[q], B[q,p+1], D[q,p+1]) as the kernels use them."""
    n = p + 1
    nodes, pts, w = np.zeros(n), np.zeros(q), np.zeros(q)
    B, D = np.zeros((q, n)), np.zeros((q, n))
    _check(load().elas_tables(p, q, _dptr(nodes), _dptr(pts), _dptr(w), _dptr(B), _dptr(D)), "elas_tables")
    return nodes, pts, w, B, D


def elas_create(nx, ny, nz, p, q, lam, mu, vertices=None, lengths=(1.0, 1.0, 1.0), faces=0,
                rank=0, nranks=1, nccl_id=None):
    """Returns an opaque handle (int).  lam/mu: scalars or (nz, ny, nx) arrays (GLOBAL)."""
    return elas_create_ex(nx, ny, nz, p, q, lam, mu, vertices, lengths, faces, rank, nranks, nccl_id,
                          VARIANT_AUTO)


def elas_variant(h):
    return load().elas_variant(h)


def _mesh_args(nx, ny, nz, lam, mu, vertices, lengths, faces, rank, nranks, nccl_id):
    """Marshal an elas_mesh; returns (mesh, lam array, mu array, keep-alive list)."""
    lam_a = np.ascontiguousarray(np.asarray(lam, dtype=np.float64).reshape(-1))
    mu_a = np.ascontiguousarray(np.asarray(mu, dtype=np.float64).reshape(-1))
    per_elem = int(lam_a.size > 1 or mu_a.size > 1)
    if per_elem:
        ne = nx * ny * nz
        lam_a = np.ascontiguousarray(np.broadcast_to(lam_a, (ne,)) if lam_a.size == 1 else lam_a)
        mu_a = np.ascontiguousarray(np.broadcast_to(mu_a, (ne,)) if mu_a.size == 1 else mu_a)
        if lam_a.size != ne or mu_a.size != ne:
            raise ValueError("per-element lambda/mu must have nx*ny*nz entries")
    m = elas_mesh()
    m.nx, m.ny, m.nz = nx, ny, nz
    V = None
    if vertices is not None:
        V = np.ascontiguousarray(vertices, dtype=np.float64)
        if V.size != (nx + 1) * (ny + 1) * (nz + 1) * 3:
            raise ValueError("vertices must have (nz+1)(ny+1)(nx+1)*3 entries")
        m.vertices = _dptr(V)
    m.lx, m.ly, m.lz = lengths
    m.dirichlet_faces = faces
    m.material_per_element = per_elem
    idbuf = None
    if nccl_id is not None:
        idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        m.nccl_id = ctypes.cast(idbuf, ctypes.c_void_p)
    m.rank, m.nranks = rank, nranks
    return m, lam_a, mu_a, [V, idbuf]


def elas_create_ex(nx, ny, nz, p, q, lam, mu, vertices=None, lengths=(1.0, 1.0, 1.0), faces=0,
                   rank=0, nranks=1, nccl_id=None, variant=VARIANT_AUTO):
    """elas_create with an explicit kernel variant (VARIANT_AUTO / _SIMT / _TENSOR / _THREAD / _FOLDED)."""
    lib = load()
    m, lam_a, mu_a, keep = _mesh_args(nx, ny, nz, lam, mu, vertices, lengths, faces, rank, nranks, nccl_id)
    h = lib.elas_create_ex(ctypes.byref(m), p, q, _dptr(lam_a), _dptr(mu_a), int(variant))
    if not h:
        raise ElasError(ELAS_EINVAL, f"elas_create: {elas_last_error()}")
    return h


def elas_apply(h, x, y):
    _check(load().elas_apply(h, _ptr(x), _ptr(y)), "elas_apply")


def elas_apply_add(h, x, y):
    _check(load().elas_apply_add(h, _ptr(x), _ptr(y)), "elas_apply_add")


def elas_apply_host(h, x_host, y_host):
    """x_host / y_host: contiguous float64 numpy arrays or pinned torch CPU tensors."""
    px = x_host.ctypes.data if isinstance(x_host, np.ndarray) else x_host.data_ptr()
    py = y_host.ctypes.data if isinstance(y_host, np.ndarray) else y_host.data_ptr()
    _check(load().elas_apply_host(h, px, py), "elas_apply_host")


def elas_interface_add(h, y, lo_halo, hi_halo):
    _check(load().elas_interface_add(h, _ptr(y), _ptr(lo_halo), _ptr(hi_halo)), "elas_interface_add")


def elas_destroy(h):
    if h:
        load().elas_destroy(h)


def elas_local_dofs(h):
    return load().elas_local_dofs(h)


def elas_local_zrange(h):
    b, e = ctypes.c_int32(), ctypes.c_int32()
    _check(load().elas_local_zrange(h, ctypes.byref(b), ctypes.byref(e)), "elas_local_zrange")
    return b.value, e.value


def elas_set_stream(h, stream):
    """stream: a torch.cuda.Stream, an int cudaStream_t, or None (legacy default)."""
    s = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
    _check(load().elas_set_stream(h, s), "elas_set_stream")


def elas_profile(h, enable):
    _check(load().elas_profile(h, int(bool(enable))), "elas_profile")


def elas_profile_read(h):
    """(summed apply-kernel milliseconds, number of bracketed launches) since the last read."""
    ms, n = ctypes.c_double(), ctypes.c_int64()
    _check(load().elas_profile_read(h, ctypes.byref(ms), ctypes.byref(n)), "elas_profile_read")
    return ms.value, n.value


def elas_launches_per_apply(h):
    return load().elas_launches_per_apply(h)


def voigt_c21(C6):
    """Upper triangles (row by row) of symmetric 6 x 6 Voigt matrices: (..., 6, 6) -> (..., 21)."""
    C6 = np.asarray(C6, dtype=np.float64)
    iu = np.triu_indices(6)
    return np.ascontiguousarray(C6[..., iu[0], iu[1]])


def elas_create_aniso(nx, ny, nz, p, q, C6, vertices=None, lengths=(1.0, 1.0, 1.0), faces=0):
    """Anisotropic operator; C6: (6, 6) for all elements or (nz, ny, nx, 6, 6) per element."""
    C21 = voigt_c21(C6)
    per = int(C21.ndim > 1)
    m, lam_a, mu_a, keep = _mesh_args(nx, ny, nz, 1.0, 1.0, vertices, lengths, faces, 0, 1, None)
    m.material_per_element = per
    h = load().elas_create_aniso(ctypes.byref(m), p, q, _dptr(C21.reshape(-1)))
    if not h:
        raise ElasError(ELAS_EINVAL, f"elas_create_aniso: {elas_last_error()}")
    return h


def elas_dot(h, a, b):
    out = ctypes.c_double(0.0)
    _check(load().elas_dot(h, _ptr(a), _ptr(b), ctypes.byref(out)), "elas_dot")
    return out.value


def elas_debug_checks(selftest=False):
    """(failed device bounds checks since the last call, source line of the first); debug build."""
    line = ctypes.c_int(0)
    n = load().elas_debug_checks(ctypes.byref(line), 1 if selftest else 0)
    if n < 0:
        raise ElasError(n, f"elas_debug_checks: {elas_last_error()}")
    return n, line.value


def elas_debug_build():
    return bool(load().elas_debug_build())


def elas_set_peer_exchange(h, on):
    """Collective over the op's communicator: NVLink peer-store interface sums (on) or NCCL (off)."""
    _check(load().elas_set_peer_exchange(h, 1 if on else 0), "elas_set_peer_exchange")


def elas_set_deterministic(h, on):
    _check(load().elas_set_deterministic(h, int(bool(on))), "elas_set_deterministic")


def elas_diagonal(h, d):
    _check(load().elas_diagonal(h, _ptr(d)), "elas_diagonal")


def elas_cheb_create(h, order=3, alpha=0.1, beta=1.1, power_iters=10, v0=None, seed=0):
    c = load().elas_cheb_create(h, order, alpha, beta, power_iters, _ptr(v0), seed)
    if not c:
        raise ElasError(ELAS_EINVAL, f"elas_cheb_create: {elas_last_error()}")
    return c


def elas_cheb_lambda_max(c):
    return load().elas_cheb_lambda_max(c)


def elas_cheb_apply(c, b, x):
    _check(load().elas_cheb_apply(c, _ptr(b), _ptr(x)), "elas_cheb_apply")


def elas_cheb_destroy(c):
    load().elas_cheb_destroy(c)


def elas_pcg(h, precond, cheb, b, x, rtol, maxit, history=False):
    """Returns (iterations, converged, rel_residual, history array or None)."""
    import numpy as np
    rep = elas_solve_report()
    hist = np.zeros(maxit + 1) if history else None
    _check(load().elas_pcg(h, precond, cheb, _ptr(b), _ptr(x), rtol, maxit, ctypes.byref(rep),
                           _dptr(hist) if history else None), "elas_pcg")
    return rep.iterations, bool(rep.converged), rep.rel_residual, (hist[:rep.iterations + 1] if history else None)


def elas_gmg_create(nx, ny, nz, p, q, lam, mu, vertices=None, lengths=(1.0, 1.0, 1.0), faces=0, levels=2,
                    order=3, alpha=0.1, beta=1.1, power_iters=10, seed=1, coarse_rtol=-1.0, coarse_maxit=20,
                    variant=VARIANT_AUTO, rank=0, nranks=1, nccl_id=None):
    m, lam_a, mu_a, keep = _mesh_args(nx, ny, nz, lam, mu, vertices, lengths, faces, rank, nranks, nccl_id)
    g = load().elas_gmg_create(ctypes.byref(m), p, q, _dptr(lam_a), _dptr(mu_a), levels, order, alpha, beta,
                               power_iters, seed, coarse_rtol, coarse_maxit, int(variant))
    if not g:
        raise ElasError(ELAS_EINVAL, f"elas_gmg_create: {elas_last_error()}")
    return g


def elas_gmg_level_op(g, level):
    return load().elas_gmg_level_op(g, level)


def elas_gmg_levels(g):
    return load().elas_gmg_levels(g)


def elas_gmg_set_stream(g, stream):
    s = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
    _check(load().elas_gmg_set_stream(g, s), "elas_gmg_set_stream")


def elas_gmg_apply(g, b, x):
    _check(load().elas_gmg_apply(g, _ptr(b), _ptr(x)), "elas_gmg_apply")


def elas_gmg_transfer(g, level, restrict, src, dst):
    _check(load().elas_gmg_transfer(g, level, int(restrict), _ptr(src), _ptr(dst)), "elas_gmg_transfer")


def elas_pcg_gmg(h, g, b, x, rtol, maxit, history=False):
    rep = elas_solve_report()
    hist = np.zeros(maxit + 1) if history else None
    _check(load().elas_pcg_gmg(h, g, _ptr(b), _ptr(x), rtol, maxit, ctypes.byref(rep),
                               _dptr(hist) if history else None), "elas_pcg_gmg")
    return rep.iterations, bool(rep.converged), rep.rel_residual, (hist[:rep.iterations + 1] if history else None)


def elas_gmg_destroy(g):
    load().elas_gmg_destroy(g)


# ------------------------------------------------------------------ convenience wrapper

class Operator:
    """Owns one elas_op handle.  Applies run on `stream` (default: torch's current stream)."""

    def __init__(self, nx, ny, nz, p, q, lam, mu, vertices=None, lengths=(1.0, 1.0, 1.0),
                 faces=0, rank=0, nranks=1, nccl_id=None, stream=None, variant=VARIANT_AUTO):
        self.p, self.q = p, q
        self.h = elas_create_ex(nx, ny, nz, p, q, lam, mu, vertices, lengths, faces, rank, nranks,
                                nccl_id, variant)
        self.variant = elas_variant(self.h)
        if stream is None:
            import torch
            stream = torch.cuda.current_stream()
        elas_set_stream(self.h, stream)
        self.local_dofs = elas_local_dofs(self.h)
        self.zrange = elas_local_zrange(self.h)
        self._chebs = []

    @classmethod
    def anisotropic(cls, P, C6, stream=None):
        """Operator of the general anisotropic material (Eq. 2) on the mesh of synth.Problem P."""
        self = cls.__new__(cls)
        self.p, self.q = P.p, P.q
        self.h = elas_create_aniso(P.nx, P.ny, P.nz, P.p, P.q, C6, P.vertices, (P.lx, P.ly, P.lz), P.dirichlet_faces)
        self.variant = elas_variant(self.h)
        if stream is None:
            import torch
            stream = torch.cuda.current_stream()
        elas_set_stream(self.h, stream)
        self.local_dofs = elas_local_dofs(self.h)
        self.zrange = elas_local_zrange(self.h)
        self._chebs = []
        return self

    @classmethod
    def from_problem(cls, P, rank=0, nranks=1, nccl_id=None, stream=None, variant=VARIANT_AUTO):
        """Build from a synth.Problem (affine problems pass vertices=NULL)."""
        V = None if P.vertices is None else P.vertices
        return cls(P.nx, P.ny, P.nz, P.p, P.q, P.lam, P.mu, V, (P.lx, P.ly, P.lz),
                   P.dirichlet_faces, rank, nranks, nccl_id, stream, variant)

    def apply(self, x, y):
        elas_apply(self.h, x, y)

    def apply_add(self, x, y):
        """y += A x (single GPU)."""
        elas_apply_add(self.h, x, y)

    def apply_host(self, x_host, y_host):
        elas_apply_host(self.h, x_host, y_host)

    def interface_add(self, y, lo, hi):
        elas_interface_add(self.h, y, lo, hi)

    def set_stream(self, stream):
        elas_set_stream(self.h, stream)

    def diagonal(self, d):
        elas_diagonal(self.h, d)

    def set_deterministic(self, on=True):
        elas_set_deterministic(self.h, on)

    def set_peer_exchange(self, on=True):
        """NVLink peer-store interface sums instead of NCCL send/recv (collective; NCCL slab ops)."""
        elas_set_peer_exchange(self.h, on)

    def chebyshev(self, order=3, alpha=0.1, beta=1.1, power_iters=10, v0=None, seed=0):
        c = Chebyshev(self, order, alpha, beta, power_iters, v0, seed)
        self._chebs.append(weakref.ref(c))
        return c

    def pcg(self, b, x, precond=PC_JACOBI, cheb=None, rtol=1e-8, maxit=1000, history=False):
        return elas_pcg(self.h, precond, cheb.h if cheb is not None else None, b, x, rtol, maxit, history)

    @property
    def launches_per_apply(self):
        return elas_launches_per_apply(self.h)

    def close(self):
        if self.h:
            for ref in getattr(self, "_chebs", []):   # smoothers hold the op: destroy them first
                c = ref()
                if c is not None:
                    c.close()
            elas_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Chebyshev:
    """Owns one elas_cheb handle (smoother / preconditioner of an Operator)."""

    def __init__(self, op, order=3, alpha=0.1, beta=1.1, power_iters=10, v0=None, seed=0):
        self.op = op
        self.h = elas_cheb_create(op.h, order, alpha, beta, power_iters, v0, seed)
        self.lambda_max = elas_cheb_lambda_max(self.h)

    def apply(self, b, x):
        elas_cheb_apply(self.h, b, x)

    def close(self):
        if self.h:
            elas_cheb_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GMG:
    """Owns one elas_gmg handle: the V-cycle hierarchy built from a fine mesh (C ABI
    elas_gmg_create).  `op_h` is a non-owning handle of the finest level's operator."""

    def __init__(self, nx, ny, nz, p, q, lam, mu, vertices=None, lengths=(1.0, 1.0, 1.0), faces=0, levels=2,
                 order=3, alpha=0.1, beta=1.1, power_iters=10, seed=1, coarse_rtol=-1.0, coarse_maxit=20,
                 variant=VARIANT_AUTO, stream=None, rank=0, nranks=1, nccl_id=None):
        self.h = elas_gmg_create(nx, ny, nz, p, q, lam, mu, vertices, lengths, faces, levels, order, alpha, beta,
                                 power_iters, seed, coarse_rtol, coarse_maxit, variant, rank, nranks, nccl_id)
        if stream is None:
            import torch
            stream = torch.cuda.current_stream()
        elas_gmg_set_stream(self.h, stream)
        self.levels = elas_gmg_levels(self.h)
        self.op_h = elas_gmg_level_op(self.h, 0)
        self.local_dofs = elas_local_dofs(self.op_h)

    @classmethod
    def from_problem(cls, P, **kw):
        return cls(P.nx, P.ny, P.nz, P.p, P.q, P.lam, P.mu, P.vertices, (P.lx, P.ly, P.lz), P.dirichlet_faces, **kw)

    def level_op(self, level):
        return elas_gmg_level_op(self.h, level)

    def level_dofs(self, level):
        return elas_local_dofs(self.level_op(level))

    def apply(self, b, x):
        """One V-cycle: x = M b."""
        elas_gmg_apply(self.h, b, x)

    def transfer(self, level, restrict, src, dst):
        elas_gmg_transfer(self.h, level, restrict, src, dst)

    def apply_op(self, x, y):
        """The finest-level operator: y = A x."""
        elas_apply(self.op_h, x, y)

    def pcg(self, b, x, rtol=1e-8, maxit=500, history=False):
        return elas_pcg_gmg(self.op_h, self.h, b, x, rtol, maxit, history)

    def close(self):
        if self.h:
            elas_gmg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
