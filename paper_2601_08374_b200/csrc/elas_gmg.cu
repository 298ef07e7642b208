// Geometric multigrid V-cycle on the GPU (Sec. 3 and
// Fig. 2: "a smoother, inter-grid transfer operators, and a coarse-grid solver"; "a matrix-free
// Chebyshev polynomial smoother is used" on the fine levels).  Readings R22-R25 in DESIGN.md:
//
// * hierarchy: h-coarsening by 2 per axis, same p and q; coarse vertices = fine vertices of even
//   index; coarse lambda, mu = the mean of the 8 children; same Dirichlet faces.  Every level is
//   an ordinary elas_op (the fused apply kernels), with its own Chebyshev smoother.
// * transfers: finite element interpolation in reference coordinates.  On the structured mesh
//   the prolongation is a Kronecker product P = Pz (x) Py (x) Px of 1D interpolations (fine node
//   I_f -> owning coarse element e = min(I_f / 2p, n_c - 1), offset t = I_f - 2 p e, weights
//   M[t][i] = l_i((s + xi_{t - s p}) / 2), host_prolongation_1d), applied as three 1D passes;
//   the restriction is its exact transpose R = P^T (three transposed 1D passes).
// * V-cycle: x = S(b, 0); r = b - A x (constrained rows 0); b_c = R r (constrained 0);
//   x_c = V(b_c); x += P x_c; x = S(b, x).  Coarsest: PCG preconditioned by the coarse
//   Chebyshev smoother, either to a tolerance (synchronising) or a fixed iteration count (no
//   host round trip; the default).  In the default mode the whole V-cycle (~40 launches per
//   level, mostly on tiny coarse grids) is captured once into a CUDA graph and replayed.
#include <cmath>
#include <string>
#include <vector>

#include "elas_op.h"

struct elas_gmg {
  int levels = 0, p = 0;
  std::vector<elas_op*> ops;            // finest first
  std::vector<elas_cheb*> chebs;        // one per level (coarsest: the PCG preconditioner)
  std::vector<double*> vb, vx, vr;      // per level: rhs, solution (levels >= 1), residual
  std::vector<double*> ta, tb;          // per level (but the coarsest): transfer temporaries
  double* M1 = nullptr;                 // (2p+1) x (p+1) interpolation weights
  double coarse_rtol = -1.0;
  int coarse_maxit = 20;
  // CUDA graph of one V-cycle (fixed-length coarse solve => no host synchronisation inside), for
  // the (b, x) pointers it was captured with; replayed on a private stream ordered after/before
  // the ops' stream by events (the legacy default stream cannot be captured)
  cudaStream_t gstream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaGraphExec_t gexec = nullptr;
  const double* gb = nullptr;
  double* gx = nullptr;
};

namespace elas {
namespace {

int gfail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? ELAS_ENOMEM : ELAS_ECUDA;
}
#define GK(expr, what)                               \
  do {                                               \
    cudaError_t e_ = (expr);                         \
    if (e_ != cudaSuccess) return gfail(e_, what);   \
  } while (0)

int gblocks(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return (int)(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

struct Dims {
  int64_t d[3];
};

// out (dims `od`, 3 components) = 1D prolongation along `axis` of `in` (same dims but the axis,
// which has nc p + 1 coarse nodes)
__global__ void prolong_axis_kernel(const double* __restrict__ in, double* __restrict__ out, Dims od, int axis,
                                    const double* __restrict__ M, int p, int nc) {
  const int64_t n0 = od.d[0], n1 = od.d[1], n2 = od.d[2];
  const int64_t total = 3 * n0 * n1 * n2;
  int64_t id[3] = {n0, n1, n2};
  id[axis] = (int64_t)nc * p + 1;                       // input extent along the axis
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t;
    int64_t i[3];
    i[0] = r % n0; r /= n0;
    i[1] = r % n1; r /= n1;
    i[2] = r % n2;
    const int64_t c = r / n2;
    const int64_t If = i[axis];
    int64_t e = If / (2 * p);
    if (e > nc - 1) e = nc - 1;
    const int tt = (int)(If - 2 * p * e);
    int64_t j[3] = {i[0], i[1], i[2]};
    double acc = 0.0;
    for (int k = 0; k <= p; ++k) {
      j[axis] = e * p + k;
      acc = fma(M[tt * (p + 1) + k], in[j[0] + id[0] * (j[1] + id[1] * (j[2] + id[2] * c))], acc);
    }
    out[t] = acc;
  }
}

// out (dims `od`, axis extent nc p + 1) = transposed 1D prolongation along `axis` of `in`
// (axis extent 2 nc p + 1): out[I_c] = sum over the fine nodes I_f owned by an element containing
// I_c of M[t][i] in[I_f]
// skip0: leave out fine index 0 along the axis (a slab's lower interface plane, owned by the rank
// below, whose restriction already counts it)
__global__ void restrict_axis_kernel(const double* __restrict__ in, double* __restrict__ out, Dims od, int axis,
                                     const double* __restrict__ M, int p, int nc, int skip0) {
  const int64_t n0 = od.d[0], n1 = od.d[1], n2 = od.d[2];
  const int64_t total = 3 * n0 * n1 * n2;
  int64_t id[3] = {n0, n1, n2};
  id[axis] = 2 * (int64_t)nc * p + 1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t;
    int64_t i[3];
    i[0] = r % n0; r /= n0;
    i[1] = r % n1; r /= n1;
    i[2] = r % n2;
    const int64_t c = r / n2;
    const int64_t Ic = i[axis];
    int64_t j[3] = {i[0], i[1], i[2]};
    double acc = 0.0;
    for (int64_t e = Ic / p - 1; e <= Ic / p; ++e) {
      if (e < 0 || e >= nc) continue;
      const int k = (int)(Ic - e * p);
      if (k < 0 || k > p) continue;
      const int tmax = (e == nc - 1) ? 2 * p : 2 * p - 1;      // the owner rule of the prolongation
      for (int tt = (skip0 && e == 0) ? 1 : 0; tt <= tmax; ++tt) {
        j[axis] = 2 * p * e + tt;
        acc = fma(M[tt * (p + 1) + k], in[j[0] + id[0] * (j[1] + id[1] * (j[2] + id[2] * c))], acc);
      }
    }
    out[t] = acc;
  }
}

__device__ __forceinline__ bool cons_node_g(int64_t node, const Slab& s) {
  const int I = (int)(node % s.Nx), J = (int)((node / s.Nx) % s.Ny), K = (int)(node / ((int64_t)s.Nx * s.Ny));
  const uint32_t f = s.faces;
  return ((f & ELAS_FACE_XMIN) && I == 0) || ((f & ELAS_FACE_XMAX) && I == s.Nx - 1) ||
         ((f & ELAS_FACE_YMIN) && J == 0) || ((f & ELAS_FACE_YMAX) && J == s.Ny - 1) ||
         ((f & ELAS_FACE_ZMIN) && K == 0) || ((f & ELAS_FACE_ZMAX) && K == s.Nz - 1);
}

// r = b - Ax on free rows, 0 on constrained rows
__global__ void residual_kernel(const double* __restrict__ b, double* __restrict__ r, Slab s) {
  const int64_t n = 3 * s.nodes;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    r[t] = (s.faces && cons_node_g(t % s.nodes, s)) ? 0.0 : b[t] - r[t];
}

__global__ void mask_kernel(double* __restrict__ v, Slab s) {
  const int64_t n = 3 * s.nodes;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    if (cons_node_g(t % s.nodes, s)) v[t] = 0.0;
}

// x += c on free rows
__global__ void add_correction_kernel(double* __restrict__ x, const double* __restrict__ c, Slab s) {
  const int64_t n = 3 * s.nodes;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    if (!(s.faces && cons_node_g(t % s.nodes, s))) x[t] += c[t];
}

// fine (level l) -> coarse (level l+1): x, then y, then z
int restrict_to(elas_gmg* g, int l, const double* fine, double* coarse) {
  const Slab& f = g->ops[l]->slab;
  const Slab& c = g->ops[l + 1]->slab;
  cudaStream_t st = g->ops[l]->stream;
  const int p = g->p;
  Dims d1{{c.Nx, f.Ny, f.Nz}}, d2{{c.Nx, c.Ny, f.Nz}}, d3{{c.Nx, c.Ny, c.Nz}};
  // z-slabs: the fine vector is replicated on the interface planes; only the owner (the rank below)
  // counts a shared fine plane, and the coarse interface planes are then summed over the
  // neighbours like the apply's (exchange_planes; the caller does it in external mode)
  const int skip0 = g->ops[l]->rank > 0 ? 1 : 0;
  restrict_axis_kernel<<<gblocks(3 * d1.d[0] * d1.d[1] * d1.d[2]), 256, 0, st>>>(fine, g->ta[l], d1, 0, g->M1, p, c.nx, 0);
  restrict_axis_kernel<<<gblocks(3 * d2.d[0] * d2.d[1] * d2.d[2]), 256, 0, st>>>(g->ta[l], g->tb[l], d2, 1, g->M1, p, c.ny, 0);
  restrict_axis_kernel<<<gblocks(3 * d3.d[0] * d3.d[1] * d3.d[2]), 256, 0, st>>>(g->tb[l], coarse, d3, 2, g->M1, p, c.nz,
                                                                                skip0);
  GK(cudaGetLastError(), "restriction kernels");
  int rc;
  if ((rc = exchange_planes(g->ops[l + 1], coarse))) return rc;
  if (c.faces) mask_kernel<<<gblocks(3 * c.nodes), 256, 0, st>>>(coarse, c);
  GK(cudaGetLastError(), "restriction mask");
  return ELAS_OK;
}

// coarse (level l+1) -> fine (level l)
int prolong_to(elas_gmg* g, int l, const double* coarse, double* fine) {
  const Slab& f = g->ops[l]->slab;
  const Slab& c = g->ops[l + 1]->slab;
  cudaStream_t st = g->ops[l]->stream;
  const int p = g->p;
  Dims d1{{f.Nx, c.Ny, c.Nz}}, d2{{f.Nx, f.Ny, c.Nz}}, d3{{f.Nx, f.Ny, f.Nz}};
  prolong_axis_kernel<<<gblocks(3 * d1.d[0] * d1.d[1] * d1.d[2]), 256, 0, st>>>(coarse, g->ta[l], d1, 0, g->M1, p, c.nx);
  prolong_axis_kernel<<<gblocks(3 * d2.d[0] * d2.d[1] * d2.d[2]), 256, 0, st>>>(g->ta[l], g->tb[l], d2, 1, g->M1, p, c.ny);
  prolong_axis_kernel<<<gblocks(3 * d3.d[0] * d3.d[1] * d3.d[2]), 256, 0, st>>>(g->tb[l], fine, d3, 2, g->M1, p, c.nz);
  GK(cudaGetLastError(), "prolongation kernels");
  return ELAS_OK;
}

int vcycle(elas_gmg* g, int l, const double* b, double* x) {
  elas_op* op = g->ops[l];
  int rc;
  if (l == g->levels - 1) {
    elas_cheb* ch = g->chebs[l];
    const bool check = g->coarse_rtol > 0.0;
    return pcg_core(op, PC_CALLBACK, [ch](const double* r, double* z) { return cheb_run(ch, r, z, true); }, b, x,
                    check ? g->coarse_rtol : 0.0, g->coarse_maxit, check, nullptr, nullptr);
  }
  const Slab& s = op->slab;
  cudaStream_t st = op->stream;
  double* r = g->vr[l];
  if ((rc = cheb_run(g->chebs[l], b, x, true))) return rc;           // pre-smoothing from x = 0
  if ((rc = elas_apply(op, x, r))) return rc;
  residual_kernel<<<gblocks(3 * s.nodes), 256, 0, st>>>(b, r, s);
  GK(cudaGetLastError(), "residual kernel");
  if ((rc = restrict_to(g, l, r, g->vb[l + 1]))) return rc;
  if ((rc = vcycle(g, l + 1, g->vb[l + 1], g->vx[l + 1]))) return rc;
  if ((rc = prolong_to(g, l, g->vx[l + 1], r))) return rc;
  add_correction_kernel<<<gblocks(3 * s.nodes), 256, 0, st>>>(x, r, s);
  GK(cudaGetLastError(), "correction kernel");
  return cheb_run(g->chebs[l], b, x, false);                          // post-smoothing
}

int vcycle_graph(elas_gmg* g, const double* b, double* x) {
  if (g->coarse_rtol > 0.0) return vcycle(g, 0, b, x);        // synchronising coarse solve: eager
  if (g->ops[0]->nranks > 1) return vcycle(g, 0, b, x);       // z-slabs (NCCL inside): eager
  cudaStream_t user = g->ops[0]->stream;
  int rc;
  if (!g->gexec || g->gb != b || g->gx != x) {
    if (g->gexec) { cudaGraphExecDestroy(g->gexec); g->gexec = nullptr; }
    if ((rc = vcycle(g, 0, b, x))) return rc;                 // eager run: first-launch setup outside capture
    GK(cudaStreamSynchronize(user), "cudaStreamSynchronize");
    for (auto* o : g->ops) o->stream = g->gstream;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamBeginCapture(g->gstream, cudaStreamCaptureModeThreadLocal);
    rc = e ? gfail(e, "cudaStreamBeginCapture") : vcycle(g, 0, b, x);
    cudaError_t e2 = cudaStreamEndCapture(g->gstream, &graph);
    for (auto* o : g->ops) o->stream = user;
    if (rc) { if (graph) cudaGraphDestroy(graph); return rc; }
    GK(e2, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&g->gexec, graph, 0);
    cudaGraphDestroy(graph);
    GK(e, "cudaGraphInstantiate");
    g->gb = b;
    g->gx = x;
    return ELAS_OK;                                             // the eager run produced x
  }
  GK(cudaEventRecord(g->ev_in, user), "cudaEventRecord");
  GK(cudaStreamWaitEvent(g->gstream, g->ev_in, 0), "cudaStreamWaitEvent");
  GK(cudaGraphLaunch(g->gexec, g->gstream), "cudaGraphLaunch");
  GK(cudaEventRecord(g->ev_out, g->gstream), "cudaEventRecord");
  GK(cudaStreamWaitEvent(user, g->ev_out, 0), "cudaStreamWaitEvent");
  return ELAS_OK;
}

void free_gmg(elas_gmg* g) {
  if (!g) return;
  if (g->gexec) cudaGraphExecDestroy(g->gexec);
  if (g->gstream) cudaStreamDestroy(g->gstream);
  if (g->ev_in) cudaEventDestroy(g->ev_in);
  if (g->ev_out) cudaEventDestroy(g->ev_out);
  for (auto* c : g->chebs) elas_cheb_destroy(c);
  for (auto* o : g->ops) elas_destroy(o);
  for (auto* v : {&g->vb, &g->vx, &g->vr, &g->ta, &g->tb})
    for (double* ptr : *v) cudaFree(ptr);
  cudaFree(g->M1);
  delete g;
}

}  // namespace
}  // namespace elas

extern "C" {

elas_gmg* elas_gmg_create(const elas_mesh* fine, int p, int q, const double* lambda, const double* mu, int levels,
                          int order, double alpha, double beta, int power_iters, unsigned long long seed,
                          double coarse_rtol, int coarse_maxit, int variant) {
  using elas::set_error;
  if (!fine || !lambda || !mu) { set_error("elas_gmg_create: NULL argument"); return nullptr; }
  // levels >= 2: with one level the coarse solve would run on the finest op and share its PCG
  // work vectors and scalar slots with the outer elas_pcg_gmg iteration
  if (levels < 2 || coarse_maxit < 1) { set_error("elas_gmg_create: need levels >= 2 and coarse_maxit >= 1"); return nullptr; }
  const int f = 1 << (levels - 1);
  if (fine->nranks > 1 && fine->nz % (fine->nranks * f)) {
    set_error("elas_gmg_create: z-slabs need nz divisible by nranks * 2^(levels-1) (aligned slabs on every level)");
    return nullptr;
  }
  if (fine->nx % f || fine->ny % f || fine->nz % f) {
    set_error("elas_gmg_create: nx, ny, nz must be divisible by 2^(levels-1)");
    return nullptr;
  }
  elas_gmg* g = new elas_gmg();
  g->levels = levels;
  g->p = p;
  g->coarse_rtol = coarse_rtol;
  g->coarse_maxit = coarse_maxit;
  // host-side hierarchy: vertices (even indices), element-mean material
  elas_mesh m = *fine;
  std::vector<double> V, lam(lambda, lambda + (fine->material_per_element ? (size_t)fine->nx * fine->ny * fine->nz : 1)),
      muv(mu, mu + lam.size());
  if (fine->vertices)
    V.assign(fine->vertices, fine->vertices + (size_t)(fine->nx + 1) * (fine->ny + 1) * (fine->nz + 1) * 3);
  for (int l = 0; l < levels; ++l) {
    m.vertices = fine->vertices ? V.data() : nullptr;
    m.nccl_id = l == 0 ? fine->nccl_id : nullptr;   // coarser slab levels borrow the finest communicator
    elas_op* op = elas_create_ex(&m, p, q, lam.data(), muv.data(), variant);
    if (!op) { elas::free_gmg(g); return nullptr; }
    g->ops.push_back(op);
    if (l > 0 && fine->nccl_id && fine->nranks > 1 && elas::attach_comm(op, g->ops[0]->comm)) {
      elas::free_gmg(g);
      return nullptr;
    }
    if (l == levels - 1) break;
    // next level
    const int nx = m.nx / 2, ny = m.ny / 2, nz = m.nz / 2;
    if (fine->vertices) {
      std::vector<double> W((size_t)(nx + 1) * (ny + 1) * (nz + 1) * 3);
      for (int k = 0; k <= nz; ++k)
        for (int j = 0; j <= ny; ++j)
          for (int i = 0; i <= nx; ++i)
            for (int c = 0; c < 3; ++c)
              W[(((size_t)k * (ny + 1) + j) * (nx + 1) + i) * 3 + c] =
                  V[(((size_t)(2 * k) * (m.ny + 1) + 2 * j) * (m.nx + 1) + 2 * i) * 3 + c];
      V.swap(W);
    }
    if (fine->material_per_element) {
      std::vector<double> L2((size_t)nx * ny * nz), M2((size_t)nx * ny * nz);
      for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
          for (int i = 0; i < nx; ++i) {
            double a = 0.0, b = 0.0;
            for (int dk = 0; dk < 2; ++dk)
              for (int dj = 0; dj < 2; ++dj)
                for (int di = 0; di < 2; ++di) {
                  const size_t e = ((size_t)(2 * k + dk) * m.ny + (2 * j + dj)) * m.nx + (2 * i + di);
                  a += lam[e];
                  b += muv[e];
                }
            L2[((size_t)k * ny + j) * nx + i] = 0.125 * a;
            M2[((size_t)k * ny + j) * nx + i] = 0.125 * b;
          }
      lam.swap(L2);
      muv.swap(M2);
    }
    m.nx = nx;
    m.ny = ny;
    m.nz = nz;
  }
  // smoothers (and the coarse preconditioner) + work vectors
  // (external-exchange slabs: transfers only, no smoothers -- their dots cannot be reduced)
  for (int l = 0; l < levels && !g->ops[0]->external; ++l) {
    elas_cheb* ch = elas_cheb_create(g->ops[l], order, alpha, beta, power_iters, nullptr, seed);
    if (!ch) { elas::free_gmg(g); return nullptr; }
    g->chebs.push_back(ch);
  }
  if (cudaStreamCreateWithFlags(&g->gstream, cudaStreamNonBlocking) ||
      cudaEventCreateWithFlags(&g->ev_in, cudaEventDisableTiming) ||
      cudaEventCreateWithFlags(&g->ev_out, cudaEventDisableTiming)) {
    set_error("elas_gmg_create: stream/event creation failed");
    elas::free_gmg(g);
    return nullptr;
  }
  std::vector<double> Mh((size_t)(2 * p + 1) * (p + 1));
  elas::host_prolongation_1d(p, Mh.data());
  cudaError_t e = cudaMalloc(&g->M1, sizeof(double) * Mh.size());
  if (!e) e = cudaMemcpy(g->M1, Mh.data(), sizeof(double) * Mh.size(), cudaMemcpyHostToDevice);
  for (int l = 0; l < levels && !e; ++l) {
    const elas::Slab& s = g->ops[l]->slab;
    const size_t nb = sizeof(double) * 3 * (size_t)s.nodes;
    double *vb = nullptr, *vx = nullptr, *vr = nullptr, *ta = nullptr, *tb = nullptr;
    if (l > 0) {
      if (!e) e = cudaMalloc(&vb, nb);
      if (!e) e = cudaMalloc(&vx, nb);
    }
    if (l < levels - 1) {
      const elas::Slab& c = g->ops[l + 1]->slab;
      const size_t a1 = 3 * (size_t)std::max((int64_t)c.Nx * s.Ny * s.Nz, (int64_t)s.Nx * c.Ny * c.Nz);
      const size_t a2 = 3 * (size_t)std::max((int64_t)c.Nx * c.Ny * s.Nz, (int64_t)s.Nx * s.Ny * c.Nz);
      if (!e) e = cudaMalloc(&vr, nb);
      if (!e) e = cudaMalloc(&ta, sizeof(double) * a1);
      if (!e) e = cudaMalloc(&tb, sizeof(double) * a2);
    }
    g->vb.push_back(vb);
    g->vx.push_back(vx);
    g->vr.push_back(vr);
    g->ta.push_back(ta);
    g->tb.push_back(tb);
  }
  if (e) {
    elas::gfail(e, "elas_gmg_create allocations");
    elas::free_gmg(g);
    return nullptr;
  }
  return g;
}

elas_op* elas_gmg_level_op(elas_gmg* g, int level) {
  if (!g || level < 0 || level >= g->levels) return nullptr;
  return g->ops[level];
}

int elas_gmg_levels(const elas_gmg* g) { return g ? g->levels : -1; }

int elas_gmg_set_stream(elas_gmg* g, void* stream) {
  if (!g) { elas::set_error("elas_gmg_set_stream: NULL"); return ELAS_EINVAL; }
  for (auto* o : g->ops) elas_set_stream(o, stream);
  if (g->gexec) { cudaGraphExecDestroy(g->gexec); g->gexec = nullptr; }
  return ELAS_OK;
}

int elas_gmg_transfer(elas_gmg* g, int level, int restrict_, const double* in, double* out) {
  if (!g || !in || !out || level < 0 || level >= g->levels - 1) {
    elas::set_error("elas_gmg_transfer: NULL argument or level outside [0, levels-1)");
    return ELAS_EINVAL;
  }
  return restrict_ ? elas::restrict_to(g, level, in, out) : elas::prolong_to(g, level, in, out);
}

int elas_gmg_apply(elas_gmg* g, const double* b, double* x) {
  if (!g || !b || !x) { elas::set_error("elas_gmg_apply: NULL argument"); return ELAS_EINVAL; }
  if (b == x) { elas::set_error("elas_gmg_apply: b and x must not alias"); return ELAS_EINVAL; }
  if (g->ops[0]->external) {
    elas::set_error("elas_gmg_apply: external-exchange slabs support transfers only (the V-cycle needs NCCL)");
    return ELAS_EINVAL;
  }
  return elas::vcycle_graph(g, b, x);
}

int elas_pcg_gmg(elas_op* op, elas_gmg* g, const double* b, double* x, double rtol, int maxit,
                 elas_solve_report* rep, double* history) {
  if (!op || !g || !b || !x) { elas::set_error("elas_pcg_gmg: NULL argument"); return ELAS_EINVAL; }
  if (op->nranks != g->ops[0]->nranks || op->rank != g->ops[0]->rank || op->external || g->ops[0]->external ||
      g->ops[0]->slab.nodes != op->slab.nodes || g->ops[0]->stream != op->stream) {
    elas::set_error("elas_pcg_gmg: the V-cycle's finest level must match op (slab, vector length, stream; NCCL mode)");
    return ELAS_EINVAL;
  }
  if (b == x || maxit < 0 || !(rtol >= 0.0)) { elas::set_error("elas_pcg_gmg: need b != x, maxit >= 0, rtol >= 0"); return ELAS_EINVAL; }
  // flexible CG unless the coarse solve converges to a tolerance (then M is a fixed linear map)
  return elas::pcg_core(op, elas::PC_CALLBACK, [g](const double* r, double* z) { return elas::vcycle_graph(g, r, z); }, b,
                        x, rtol, maxit, true, rep, history, !(g->coarse_rtol > 0.0));
}

void elas_gmg_destroy(elas_gmg* g) {
  if (g && !g->ops.empty()) cudaStreamSynchronize(g->ops[0]->stream);
  elas::free_gmg(g);
}

}  // extern "C"
