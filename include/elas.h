/*
 * elas.h -- C ABI of libelas.so: the matrix-free (partial-assembly) action y = A x of the
 * 3D linear-elasticity stiffness operator on tensor-product Q_p hexahedra, FP64, on B200.
 *
 * What the operator is (citations are to the paper text, /root/reference/PAPER.md):
 *   - Hooke's law sigma = lambda (div u) I + 2 mu eps(u)                  PAPER.md:147-150, Eq. 3
 *   - bilinear form a(u,v) = int sigma(u) : grad v                         PAPER.md:152-156, Eq. 4
 *   - A_ij = a(phi_i, phi_j) (Galerkin system A U = F)                     PAPER.md:158-162, Eq. 5
 *   - A = P^T G^T B^T D B G P applied on the fly (partial assembly)
 *   - tensor-product basis + sum factorisation, O(p^4) per element
 *   - one element-centric fused pass (macro-kernel fusion, Alg. 2)
 *   - Voigt-symmetric stress at the quadrature points (Sec. 4.3, Eq. 6)
 * Discretisation readings (where the paper is silent) are listed in DESIGN.md section 3:
 * Lagrange basis on Gauss-Lobatto-Legendre nodes, q-point Gauss-Legendre quadrature per
 * direction, trilinear geometry, reference cube [0,1]^3.
 *
 * Mesh and vector conventions (R6):
 *   - structured nx x ny x nz grid of trilinear hexahedra, vertex (i,j,k) at
 *     vertices[((k*(ny+1) + j)*(nx+1) + i)*3 + {0,1,2}]  (x fastest);
 *   - global node (I,J,K), I in [0, nx p], id = I + Nx (J + Ny K), Nx = nx p + 1, ...;
 *   - vectors are component-blocked: dof = c N + id, c = 0,1,2 (all x, then y, then z).
 *
 * Multi-GPU (one process per GPU): the element grid is split into contiguous z-slabs,
 * rank r owning element layers ez in [floor(r nz / P), floor((r+1) nz / P)).  Rank r holds
 * node planes K in [ez_begin p, ez_end p] (both ends): interface planes are replicated and,
 * after elas_apply, both replicas hold the full sum (the P^T of PAPER.md:169).
 *
 * Error behaviour: functions return ELAS_OK (0) or a negative ELAS_E* code; elas_create
 * returns NULL.  In every failing case elas_last_error() returns a thread-local message.
 * Asynchronous CUDA faults surface at the next call that synchronises.
 */
#ifndef ELAS_H
#define ELAS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ELAS_OK 0
#define ELAS_EINVAL (-1) /* bad sizes, p not in [1,8], q not in {p+1,p+2}, NULL or misaligned
                            pointers, x == y, mu <= 0 or 3 lambda + 2 mu <= 0, or a call
                            that does not match the op's mode                        */
#define ELAS_EGEOM (-2)  /* det J <= 0 at some quadrature point                         */
#define ELAS_ENOMEM (-3) /* device or host allocation failed                            */
#define ELAS_ECUDA (-4)  /* CUDA runtime error (message has the CUDA error string)       */
#define ELAS_ENCCL (-5)  /* NCCL error (multi-GPU exchange)                             */

/* Dirichlet face bits: all three components of every node on the face are constrained. */
#define ELAS_FACE_XMIN 1u
#define ELAS_FACE_XMAX 2u
#define ELAS_FACE_YMIN 4u
#define ELAS_FACE_YMAX 8u
#define ELAS_FACE_ZMIN 16u
#define ELAS_FACE_ZMAX 32u

typedef struct elas_op elas_op; /* opaque; owned by the library */

typedef struct {
  int32_t nx, ny, nz;           /* GLOBAL elements per axis, each >= 1                      */
  const double* vertices;       /* HOST, (nz+1)(ny+1)(nx+1)*3 doubles, x fastest, xyz per
                                   vertex; NULL => uniform grid on [0,lx]x[0,ly]x[0,lz]      */
  double lx, ly, lz;            /* > 0; used only when vertices == NULL                     */
  uint32_t dirichlet_faces;     /* OR of ELAS_FACE_* ; y = Z A Z x + (I - Z) x               */
  int32_t material_per_element; /* 0: lambda, mu point to 1 value each;
                                   1: to nx*ny*nz values each (element order x fastest)     */
  const void* nccl_id;          /* NULL, or a HOST pointer to a 128-byte ncclUniqueId shared
                                   by all ranks: the library then owns an NCCL communicator
                                   and does the interface sum inside elas_apply             */
  int32_t rank, nranks;         /* nranks == 1: single GPU.  nranks > 1 and nccl_id == NULL:
                                   "external exchange" mode -- elas_apply leaves the
                                   interface planes as LOCAL partial sums and the caller
                                   completes them with elas_interface_add                   */
} elas_mesh;

/* Build the operator on the current CUDA device: validates the inputs, builds the 1D
 * tables (GLL nodes, Gauss-Legendre rule, Lagrange values/derivatives; host), copies the
 * vertices of this rank's slab to the device and runs the quadrature-data setup kernel
 * (J, det J, A = J^{-1}, W = w det J; stores A~ = sqrt(mu_e W) A per point and
 * r_e = lambda_e / mu_e per element), and writes the folded 1D tables of (p, q) into the
 * folded kernels' constant bank on the current device (identical bytes for every operator of
 * that (p, q), so concurrent creates are safe).  Synchronises.  lambda/mu: HOST pointers.
 * q must be p+1 or p+2.  Host arrays are copied; the caller may free them on return.
 * Returns NULL on error (see elas_last_error). */
elas_op* elas_create(const elas_mesh* mesh, int p, int q, const double* lambda, const double* mu);

/* General anisotropic material (Eq. 2): sigma_voigt = C eps_voigt with
 * eps_voigt = [e11, e22, e33, 2 e23, 2 e13, 2 e12].  C21: HOST, the upper
 * triangle of the symmetric 6 x 6 Voigt matrix row by row (C00 C01 .. C05 C11 .. C55), 21
 * doubles per element (mesh->material_per_element = 1, element order as lambda/mu) or 21 for
 * all.  The op runs the folded FP64 kernel with A~ = sqrt(W) J^{-1} and a 6 x 6 product per
 * point; elas_apply, elas_diagonal, Chebyshev, PCG and the deterministic mode work unchanged.
 * NULL + message on error (as elas_create; non-finite entries are ELAS_EINVAL). */
elas_op* elas_create_aniso(const elas_mesh* mesh, int p, int q, const double* C21);

/* Kernel variants of the fused apply (same operator, same results to rounding):
 *   ELAS_VARIANT_SIMT   FP64 FMA pipe, one thread per 1D fibre (every p, q);
 *   ELAS_VARIANT_TENSOR FP64 tensor cores (mma.sync f64 / DMMA), one warp per element
 *                       (p = 6, q = 8 only);
 *   ELAS_VARIANT_THREAD one thread per element, sum factorisation in registers (p = 1 only);
 *   ELAS_VARIANT_FOLDED the SIMT kernel with even-odd folded 1D contractions (every p, q;
 *                       half the sum-factorisation FMAs; same qdata layout as SIMT).  For
 *                       FP64 at p = 6..8 (non-deterministic mode, stored geometry, isotropic)
 *                       it runs as the fine-grained kernel: one element per CTA of 3 q^2
 *                       threads, one-component / one-point work items;
 *   ELAS_VARIANT_FOLDED_F32  MIXED PRECISION (PAPER.md:600 future work): the folded kernel
 *                       with FP32 quadrature data (9 floats per point), FP32 tables and FP32
 *                       arithmetic; x, y stay FP64 (converted on gather, FP64 atomics on
 *                       scatter).  Accuracy ~1e-6 relative, not the FP64 1e-12 (DESIGN.md
 *                       section 11); never chosen by AUTO.
 *   ELAS_VARIANT_FOLDED_OTF  the folded FP64 kernel with GEOMETRY ON THE FLY: no stored
 *                       quadrature data (40 doubles per element instead of 9 q^3); A~ rebuilt
 *                       at every point from the trilinear map.
 *   ELAS_VARIANT_ABL_PA, ELAS_VARIANT_ABL_SF, ELAS_VARIANT_ABL_VOIGT  the paper's ablation
 *                       stages (Table 4) on B200, for measurement: unfused
 *                       gather / gradient / pointwise / transposed-contraction / scatter
 *                       kernels with the element vectors and QVec in HBM; PA = dense O(p^6)
 *                       basis-gradient contractions (Alg. 1), SF = sum factorisation (C1),
 *                       VOIGT = SF + 6-component stress in QVec (C2).  "+ fusion" (C3) and
 *                       "+ loop structure" are ELAS_VARIANT_SIMT and ELAS_VARIANT_FOLDED.  Same
 *                       results to rounding; scratch of (6 n^3 + 9 q^3) doubles per element is
 *                       allocated at the first apply.  No deterministic
 *                       mode.
 *   ELAS_VARIANT_AUTO   the faster measured variant for (p, q).
 * The choice fixes the quadrature-data layout, so it is made at creation. */
#define ELAS_VARIANT_AUTO 0
#define ELAS_VARIANT_SIMT 1
#define ELAS_VARIANT_TENSOR 2
#define ELAS_VARIANT_THREAD 3
#define ELAS_VARIANT_FOLDED 4
#define ELAS_VARIANT_FOLDED_F32 5
#define ELAS_VARIANT_FOLDED_OTF 6
#define ELAS_VARIANT_ABL_PA 7
#define ELAS_VARIANT_ABL_SF 8
#define ELAS_VARIANT_ABL_VOIGT 9

/* elas_create with an explicit kernel variant; NULL + ELAS_EINVAL message if the variant
 * does not exist for (p, q). */
elas_op* elas_create_ex(const elas_mesh* mesh, int p, int q, const double* lambda, const double* mu,
                        int variant);

/* Bitwise-reproducible applies: on != 0 splits the apply into
 * 8 launches, one per element color (parity per axis) in a fixed order; no two elements of a
 * color share a node, so every node gets one contribution per launch and the sum order is fixed.  Folded
 * variants only (ELAS_EINVAL otherwise).  Same result to rounding; y identical run to run. */
int elas_set_deterministic(elas_op* op, int on);

/* The resolved variant of an op (ELAS_VARIANT_SIMT, _TENSOR, _THREAD, _FOLDED or _FOLDED_F32), -1 if NULL. */
int elas_variant(const elas_op* op);

/* y = A x (overwrite), or y = Z A Z x + (I - Z) x with Dirichlet faces.
 * x, y: DEVICE pointers on the op's device, elas_local_dofs(op) doubles each, component-
 * blocked over this rank's node planes, 8-byte aligned, not aliased.  Asynchronous on the
 * op's stream (see elas_set_stream).  A distributed op owns halo buffers: serialise its
 * applies.  Returns ELAS_OK or ELAS_EINVAL / ELAS_ECUDA / ELAS_ENCCL. */
int elas_apply(elas_op* op, const double* x, double* y);

/* Accumulating apply y += A x (A as elas_apply applies it: y_c += x_c on constrained dofs), the
 * semantics of SPEC.md's CPU program (y += A x) for smoothers that compose
 * updates.  Single-GPU operators only (ELAS_EINVAL for nranks > 1).  Same layout, alignment,
 * aliasing and stream rules as elas_apply. */
int elas_apply_add(elas_op* op, const double* x, double* y);

/* End-to-end form of elas_apply: x_host, y_host are HOST pointers (pinned recommended);
 * copies x to an op-owned device buffer, applies, copies y back, and synchronises the
 * op's stream.  Returns as elas_apply (ELAS_ENOMEM if the staging buffers fail). */
int elas_apply_host(elas_op* op, const double* x_host, double* y_host);

/* External-exchange mode only (nranks > 1, nccl_id == NULL): add the neighbours' partial
 * interface planes into y on the op's stream.  lo_halo: the partial plane of rank r-1 for
 * the plane K = ez_begin p (NULL on rank 0); hi_halo: the partial plane of rank r+1 for
 * K = ez_end p (NULL on the last rank).  Each is 3 * Nx * Ny doubles, component-blocked,
 * DEVICE pointers.  Constrained (Dirichlet) rows are left untouched.  Returns ELAS_OK,
 * ELAS_EINVAL or ELAS_ECUDA. */
int elas_interface_add(elas_op* op, double* y, const double* lo_halo, const double* hi_halo);

/* Release everything the op owns (device memory, communicator, streams).  NULL-safe. */
void elas_destroy(elas_op* op);

/* Length of x and y on this rank: 3 * Nx * Ny * (nz_local p + 1).  -1 if op == NULL. */
int64_t elas_local_dofs(const elas_op* op);

/* This rank's element-layer range [ez_begin, ez_end).  ELAS_OK or ELAS_EINVAL. */
int elas_local_zrange(const elas_op* op, int32_t* ez_begin, int32_t* ez_end);

/* Make subsequent applies run on `cuda_stream` (a cudaStream_t; NULL = legacy default). */
int elas_set_stream(elas_op* op, void* cuda_stream);

/* Number of kernel launches one elas_apply issues (for the bench's launch accounting): the fused
 * apply (8 in colored mode, per element range), the Dirichlet-face copy when faces are
 * constrained, and the interface plane adds in NCCL mode; the y memset is not a kernel. */
int elas_launches_per_apply(const elas_op* op);

/* Measurement hook (used by bench.py): enabling starts a fresh window; while enabled, every launch of the fused apply
 * kernel inside elas_apply is bracketed by CUDA events on the op's stream.
 * elas_profile_read synchronises on the last event, returns the summed kernel time (ms) and
 * the number of bracketed launches since the previous read, and resets the counters.
 * Both return ELAS_OK, ELAS_EINVAL or ELAS_ECUDA. */
int elas_profile(elas_op* op, int enable);
int elas_profile_read(elas_op* op, double* apply_kernel_ms, int64_t* launches);

/* Solver layer: the consumers of the apply in the paper's solver (
 * PAPER.md:202-210 Sec. 3.1 "Chebyshev polynomial smoother ... the action of the matrix
 * operator A and an estimate of the operator's spectral radius ... a few Lanczos or power
 * iterations"; PAPER.md:164 CG).  Readings R18-R21 in DESIGN.md.  All vectors are DEVICE
 * pointers of elas_local_dofs(op) doubles, 8-byte aligned, on the op's stream. ----------- */

/* d = diag(Z A Z + (I - Z)): the diagonal of the operator elas_apply applies (constrained
 * rows 1), by a sum-factorised setup kernel (one CTA per element, 6 x 3 contracted q^3
 * tensors).  Multi-GPU: as elas_apply (NCCL mode sums the interface planes; external mode
 * leaves partial planes for elas_interface_add).  ELAS_OK / ELAS_EINVAL / ELAS_ECUDA. */
int elas_diagonal(elas_op* op, double* d);

/* Chebyshev smoother on D^{-1} A (D = elas_diagonal), single-GPU operators or NCCL slab mode
 * (dots allreduced; external-exchange ops are rejected).
 * Create: computes and caches D^{-1} in the op, runs `power_iters` power iterations
 *   v <- v/|v|; w = D^{-1} A v; lam = v.w; v <- w/|w|
 * from v0 (DEVICE, NULL => splitmix64 counter generator with `seed`, the same generator as
 * synth.splitmix_uniform) and sets lam_max = 1.1 lam.  The polynomial is the degree-`order`
 * Chebyshev polynomial for the interval [alpha lam_max, beta lam_max] (SPEC defaults 3, 0.1,
 * 1.1).  NULL + ELAS_EINVAL message on bad arguments (order < 1, !(0 < alpha < beta),
 * power_iters < 1, external-exchange op) or a non-positive estimate.  Owns 3 work vectors. */
typedef struct elas_cheb elas_cheb;
elas_cheb* elas_cheb_create(elas_op* op, int order, double alpha, double beta, int power_iters, const double* v0,
                            unsigned long long seed);
/* 1.1 x the power-iteration estimate (-1 if NULL). */
double elas_cheb_lambda_max(const elas_cheb* ch);
/* One smoothing pass: x <- x + p_k(D^{-1} A) D^{-1} (b - A x), classical three-term Chebyshev
 * iteration (order applies of the operator).  b, x must not alias.  Asynchronous. */
int elas_cheb_apply(elas_cheb* ch, const double* b, double* x);
void elas_cheb_destroy(elas_cheb* ch);   /* NULL-safe; synchronises the op's stream */

/* Preconditioned conjugate gradients from x = 0 (single GPU or NCCL slab mode).  precond:
 * ELAS_PC_NONE, ELAS_PC_JACOBI (D^{-1}, cached in the op) or ELAS_PC_CHEBYSHEV (z =
 * p_k(D^{-1}A) D^{-1} r with `cheb`'s operator, which may be another op of the same mesh and
 * stream -- e.g. an ELAS_VARIANT_FOLDED_F32 op: FP64 CG with a mixed-precision smoother).  Stops when sqrt(r.z / r0.z0) <= rtol or after
 * maxit iterations (not an error: report.converged = 0).  history (HOST, maxit + 1 doubles or
 * NULL) receives sqrt(r_i.z_i / r0.z0).  Synchronises once per iteration (8-byte read of r.z).
 * Dots are deterministic (fixed two-pass reduction order).  ELAS_OK / ELAS_EINVAL (bad
 * arguments, preconditioner not positive) / ELAS_ECUDA. */
#define ELAS_PC_NONE 0
#define ELAS_PC_JACOBI 1
#define ELAS_PC_CHEBYSHEV 2
typedef struct {
  int iterations;       /* iterations performed                                         */
  int converged;        /* 1 if rel_residual <= rtol                                    */
  double rel_residual;  /* sqrt(r.z / r0.z0) at exit                                     */
} elas_solve_report;
int elas_pcg(elas_op* op, int precond, elas_cheb* cheb, const double* b, double* x, double rtol, int maxit,
             elas_solve_report* report, double* history);

/* Distributed dot product a.b over the dofs this rank OWNS (the lower interface plane of a slab
 * belongs to the rank below), allreduced over the communicator in NCCL mode; in external-
 * exchange mode the rank-local partial (the caller sums them).  Synchronises; result on the
 * host.  This is the reduction elas_pcg and the power iteration use. */
int elas_dot(elas_op* op, const double* a, const double* b, double* result);

/* NVLink peer-store interface sum (SURVEY 8(e) extra; PAPER.md:604 names the parallel exchange as
 * the next bottleneck).  COLLECTIVE over the op's NCCL communicator: every rank calls it with the
 * same `on`.  on = 1: the ranks exchange CUDA IPC handles of their halo buffers and of a small
 * flag buffer with their z-neighbours (once; the mapping is kept until elas_destroy), and from
 * then on every interface sum of this op (elas_apply, elas_diagonal, the GMG restriction) copies
 * the rank's partial interface plane straight into the neighbour's halo over NVLink and
 * publishes it with a release store of the exchange epoch into the neighbour's flag; the
 * receiver's stream waits on its own flag (a one-thread spin kernel, so both GPUs must run
 * concurrently: one process per GPU) before the same plane-add as the NCCL path, then tells the
 * sender its halo may be overwritten.  Results are bitwise equal to the NCCL path.  on = 0:
 * back to NCCL send/recv.  ELAS_EINVAL for ops without a communicator (nranks == 1, external
 * mode); CUDA errors if the neighbours' memory cannot be mapped (e.g. ranks in one process). */
int elas_set_peer_exchange(elas_op* op, int on);

/* Geometric multigrid V-cycle (Sec. 3, Fig. 2).
 * Readings R22-R25 in DESIGN.md.  Z-slabs (fine->nranks > 1): nz must be divisible by
 * nranks * 2^(levels-1) so every level's slabs align (coarse slab = fine slab / 2); every level
 * is a slab op of the same rank; with fine->nccl_id the finest level owns the communicator and
 * the coarser levels borrow it, restriction counts a shared fine interface plane on the rank
 * below only and sums the coarse interface planes over NCCL, and the V-cycle runs eagerly (no
 * graph capture); without nccl_id (external-exchange mode) only elas_gmg_transfer works, and a
 * restriction leaves the coarse interface planes as LOCAL partial sums (complete them with
 * elas_interface_add on elas_gmg_level_op(g, level + 1)); apply / pcg_gmg return ELAS_EINVAL.
 * create: builds `levels` levels from `fine` (same p, q; h-coarsening by 2 per axis: nx, ny, nz
 *   divisible by 2^(levels-1); coarse vertices = fine vertices of even index; per-element
 *   lambda, mu averaged over the 8 children; same Dirichlet faces), each an elas_op of kernel
 *   `variant` (ELAS_VARIANT_AUTO or any variant valid for (p, q)) with a Chebyshev smoother
 *   (order, alpha, beta, power_iters, seed as elas_cheb_create).  Transfers: FE interpolation
 *   in reference coordinates (Kronecker product of 1D interpolations) and its transpose.
 *   Coarsest level: PCG preconditioned by its Chebyshev smoother, to coarse_rtol (> 0:
 *   synchronising convergence test) or exactly coarse_maxit iterations (coarse_rtol <= 0: no
 *   host round trip).  Host arrays are copied.  NULL + message on error.
 * create needs levels >= 2 (ELAS_EINVAL-style NULL otherwise).
 * apply: one V-cycle x = M b (x overwritten; pre- and post-smoothing with the same Chebyshev
 *   polynomial).  M is a fixed symmetric linear map only when the coarse solve converges to
 *   coarse_rtol > 0; with the default fixed-length coarse PCG (coarse_rtol <= 0) M depends on b
 *   (nonlinear), and elas_pcg_gmg then uses the flexible-CG (Polak-Ribiere) beta.  DEVICE b, x
 *   of the finest level's length; asynchronous.
 * level_op: the op of level l (0 = finest), owned by the gmg (do not destroy).
 * pcg_gmg: elas_pcg with the V-cycle as preconditioner (op: typically elas_gmg_level_op(g, 0)). */
typedef struct elas_gmg elas_gmg;
elas_gmg* elas_gmg_create(const elas_mesh* fine, int p, int q, const double* lambda, const double* mu, int levels,
                          int order, double alpha, double beta, int power_iters, unsigned long long seed,
                          double coarse_rtol, int coarse_maxit, int variant);
elas_op* elas_gmg_level_op(elas_gmg* g, int level);
int elas_gmg_levels(const elas_gmg* g);
int elas_gmg_set_stream(elas_gmg* g, void* cuda_stream);
int elas_gmg_apply(elas_gmg* g, const double* b, double* x);
/* The transfers alone: restrict_ = 0: out (level) = P in (level+1); restrict_ = 1: out (level+1)
 * = P^T in (level), constrained coarse entries zeroed.  0 <= level < levels - 1. */
int elas_gmg_transfer(elas_gmg* g, int level, int restrict_, const double* in, double* out);
int elas_pcg_gmg(elas_op* op, elas_gmg* g, const double* b, double* x, double rtol, int maxit,
                 elas_solve_report* report, double* history);
void elas_gmg_destroy(elas_gmg* g);   /* NULL-safe; synchronises */

/* Debug build (lib/libelas_debug.so, compiled with ELAS_DEBUG=1): device-side bounds checks on
 * every global gather / scatter / quadrature-data index of the apply kernels, the stand-in for
 * compute-sanitizer (closed on this pool).  A failed check is counted (it does not trap).
 * elas_debug_checks: synchronises nothing itself (call after cudaDeviceSynchronize); returns the
 * number of failed checks since the last call (>= 0; negative ELAS_E* on a CUDA error), stores
 * the source line of the first in *first_line (may be NULL) and resets the counters; selftest =
 * 1 first runs one deliberately failing check (so the debug build returns >= 1).  In the release
 * build the checks are compiled out and the count is always 0.
 * elas_debug_build: 1 in the debug build, 0 otherwise. */
int elas_debug_checks(int* first_line, int selftest);
int elas_debug_build(void);

/* Thread-local message describing the last error on this thread ("" if none). */
const char* elas_last_error(void);

/* Host-only helpers (no GPU needed) -------------------------------------------------- */

/* The slab partition: [floor(rank nz / nranks), floor((rank+1) nz / nranks)).
 * ELAS_EINVAL if nz < nranks, nranks < 1 or rank outside [0, nranks). */
int elas_slab_range(int32_t nz, int32_t rank, int32_t nranks, int32_t* ez_begin, int32_t* ez_end);

/* The 1D tables the kernels use, for inspection: nodes[p+1] (GLL on [0,1]), points[q],
 * weights[q] (Gauss-Legendre on [0,1], sum 1), B[q*(p+1)] and D[q*(p+1)] with
 * B[a*(p+1)+i] = l_i(g_a), D[a*(p+1)+i] = l_i'(g_a).  Any output may be NULL.
 * ELAS_OK or ELAS_EINVAL (p not in [1,8], q not in [1,16]). */
int elas_tables(int p, int q, double* nodes, double* points, double* weights, double* B, double* D);

/* Create a fresh 128-byte ncclUniqueId into `id_out` (host memory) on ONE rank; broadcast it
 * to the others (e.g. over a torch.distributed group) and pass it as elas_mesh.nccl_id.
 * ELAS_OK, ELAS_EINVAL (NULL) or ELAS_ENCCL. */
int elas_nccl_unique_id(void* id_out);

/* Library version (major*10000 + minor*100 + patch). */
int elas_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ELAS_H */
