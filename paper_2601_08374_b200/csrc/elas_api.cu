// The C ABI of libelas.so (include/elas.h): operator construction, apply, multi-GPU slab
// exchange over NCCL, and host-only helpers.
#include <nccl.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "elas_op.h"

#define ELAS_VERSION 10000

// AUTO picks the measured-faster variant.
#ifndef ELAS_AUTO_TENSOR
#define ELAS_AUTO_TENSOR 0   // measured: folded SIMT 30.6 vs tensor 29.8 GDoF/s at config 5
#endif
static constexpr bool kAutoTensor = ELAS_AUTO_TENSOR != 0;
#ifndef ELAS_AUTO_THREAD
#define ELAS_AUTO_THREAD 1
#endif
static constexpr bool kAutoThread = ELAS_AUTO_THREAD != 0;
// measured (tools/ab_variants.py, config 4): the folded kernel beats the plain SIMT kernel at
// every p = 2..8 (+5 % at p = 2, +19 % p = 4, +52 % p = 8)
#ifndef ELAS_AUTO_FOLDED
#define ELAS_AUTO_FOLDED 1
#endif
static constexpr bool kAutoFolded = ELAS_AUTO_FOLDED != 0;
#ifndef ELAS_HOST_CHUNKS
#define ELAS_HOST_CHUNKS 64   // z-chunks of the pipelined host apply
#endif

namespace elas {

namespace {
thread_local std::string g_err;

// per-degree dispatch (defined by ELAS_DEFINE_DEGREE in elas_apply_p<P>.cu)
}  // namespace

#define DECL(P)                                                                                  \
  cudaError_t apply_info_p##P(int q, ApplyLaunch* info);                                         \
  cudaError_t apply_launch_p##P(int q, const Slab& s, const double* x, double* y, const double* qd, \
                                const double* rr, const double* tables, int64_t e_begin,        \
                                int64_t e_end, cudaStream_t st);
DECL(1) DECL(2) DECL(3) DECL(4) DECL(5) DECL(6) DECL(7) DECL(8)
#undef DECL
#define DECL(P)                                                                                  \
  cudaError_t apply_eo_info_p##P(int q, int fp32, ApplyLaunch* info);                            \
  cudaError_t apply_eo_upload_p##P(int q, const double* fold);                                   \
  cudaError_t apply_eo_launch_p##P(int q, int fp32, const Slab& s, const double* x, double* y,   \
                                   const void* qd, const double* rr, const void* tables,        \
                                   int64_t e_begin, int64_t e_end, cudaStream_t st, const int* color, \
                                   int otf, const double* cc);
DECL(1) DECL(2) DECL(3) DECL(4) DECL(5) DECL(6) DECL(7) DECL(8)
#undef DECL

void set_error(const std::string& msg) { g_err = msg; }

cudaError_t apply_info(int p, int q, ApplyLaunch* info) {
  switch (p) {
    case 1: return apply_info_p1(q, info);
    case 2: return apply_info_p2(q, info);
    case 3: return apply_info_p3(q, info);
    case 4: return apply_info_p4(q, info);
    case 5: return apply_info_p5(q, info);
    case 6: return apply_info_p6(q, info);
    case 7: return apply_info_p7(q, info);
    case 8: return apply_info_p8(q, info);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t apply_launch(int p, int q, const Slab& s, const double* x, double* y, const double* qd,
                         const double* rr, const double* tables, int64_t e_begin, int64_t e_end,
                         cudaStream_t st) {
  switch (p) {
#define CASE(P) case P: return apply_launch_p##P(q, s, x, y, qd, rr, tables, e_begin, e_end, st);
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t apply_eo_info(int p, int q, int fp32, ApplyLaunch* info) {
  switch (p) {
#define CASE(P) case P: return apply_eo_info_p##P(q, fp32, info);
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t apply_eo_upload(int p, int q, const double* fold) {
  switch (p) {
#define CASE(P) case P: return apply_eo_upload_p##P(q, fold);
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t apply_eo_launch(int p, int q, int fp32, const Slab& s, const double* x, double* y, const void* qd,
                            const double* rr, const void* tables, int64_t e_begin, int64_t e_end,
                            cudaStream_t st, const int* color, int otf, const double* cc) {
  switch (p) {
#define CASE(P) case P: return apply_eo_launch_p##P(q, fp32, s, x, y, qd, rr, tables, e_begin, e_end, st, color, otf, cc);
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace elas

using elas::Slab;
using elas::set_error;


namespace {

int cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? ELAS_ENOMEM : ELAS_ECUDA;
}

int nccl_fail(ncclResult_t r, const char* what) {
  set_error(std::string(what) + ": " + ncclGetErrorString(r));
  return ELAS_ENCCL;
}

#define CUDA_OR(expr, what)                   \
  do {                                        \
    cudaError_t e_ = (expr);                  \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

#define NCCL_OR(expr, what)                   \
  do {                                        \
    ncclResult_t r_ = (expr);                 \
    if (r_ != ncclSuccess) return nccl_fail(r_, what); \
  } while (0)

void free_op(elas_op* op) {
  if (!op) return;
  cudaFree(op->qd);
  cudaFree(op->rr);
  cudaFree(op->tab);
  cudaFree(op->tabf);
  cudaFree(op->cc);
  cudaFree(op->xs);
  cudaFree(op->ys);
  for (void* pp : {(void*)op->peer_lo_halo, (void*)op->peer_lo_flags, (void*)op->peer_hi_halo, (void*)op->peer_hi_flags})
    if (pp) cudaIpcCloseMemHandle(pp);
  cudaFree(op->peer_flags);
  cudaFree(op->halo_lo);
  cudaFree(op->halo_hi);
  if (op->comm && !op->comm_borrowed) ncclCommDestroy(op->comm);
  if (op->comm_stream) cudaStreamDestroy(op->comm_stream);
  if (op->ev_boundary) cudaEventDestroy(op->ev_boundary);
  if (op->ev_comm) cudaEventDestroy(op->ev_comm);
  for (cudaEvent_t ev : op->prof_ev) cudaEventDestroy(ev);
  for (cudaEvent_t ev : op->host_ev) cudaEventDestroy(ev);
  cudaFree(op->abl_E);
  cudaFree(op->abl_Eo);
  cudaFree(op->abl_Q);
  cudaFree(op->abl_G);
  if (op->h2d) cudaStreamDestroy(op->h2d);
  if (op->d2h) cudaStreamDestroy(op->d2h);
  elas::free_solver_state(op);
  delete op;
}

int build(elas_op* op, const elas_mesh* m, const double* lambda, const double* mu) {
  const int p = op->p, q = op->q;
  const int nx = m->nx, ny = m->ny;
  const int nzl = op->ez1 - op->ez0;
  Slab& s = op->slab;
  s.nx = nx;
  s.ny = ny;
  s.nz = nzl;
  s.Nx = nx * p + 1;
  s.Ny = ny * p + 1;
  s.Nz = nzl * p + 1;
  s.nodes = (int64_t)s.Nx * s.Ny * s.Nz;
  uint32_t f = m->dirichlet_faces & 15u;
  if ((m->dirichlet_faces & ELAS_FACE_ZMIN) && op->rank == 0) f |= ELAS_FACE_ZMIN;
  if ((m->dirichlet_faces & ELAS_FACE_ZMAX) && op->rank == op->nranks - 1) f |= ELAS_FACE_ZMAX;
  s.faces = f;

  const int64_t ne = (int64_t)nx * ny * nzl;
  // vertices of the slab (planes ez0 .. ez1)
  const int64_t vplane = (int64_t)(nx + 1) * (ny + 1);
  std::vector<double> V((size_t)(vplane * (nzl + 1) * 3));
  for (int k = 0; k <= nzl; ++k)
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i) {
        const int64_t lv = ((int64_t)k * (ny + 1) + j) * (nx + 1) + i;
        const int64_t gv = ((int64_t)(k + op->ez0) * (ny + 1) + j) * (nx + 1) + i;
        for (int c = 0; c < 3; ++c) {
          double val;
          if (m->vertices) {
            val = m->vertices[gv * 3 + c];
          } else {
            const double L = c == 0 ? m->lx : (c == 1 ? m->ly : m->lz);
            const int n = c == 0 ? m->nx : (c == 1 ? m->ny : m->nz);
            const int idx = c == 0 ? i : (c == 1 ? j : k + op->ez0);
            val = (idx == n) ? L : idx * (L / n);
          }
          V[lv * 3 + c] = val;
        }
      }
  // material of the slab
  std::vector<double> lam((size_t)ne), muv((size_t)ne);
  const int64_t off = (int64_t)op->ez0 * nx * ny;
  for (int64_t e = 0; e < ne; ++e) {
    lam[e] = m->material_per_element ? lambda[off + e] : lambda[0];
    muv[e] = m->material_per_element ? mu[off + e] : mu[0];
    if (!(muv[e] > 0.0) || !(3.0 * lam[e] + 2.0 * muv[e] > 0.0) || !std::isfinite(lam[e])) {
      set_error("invalid material: need mu > 0 and 3 lambda + 2 mu > 0 (element " +
                std::to_string(off + e) + ")");
      return ELAS_EINVAL;
    }
  }
  // 1D tables
  const int n = p + 1;
  // tables = B | D | fold(B) | fold(D)  (the folded copies feed ELAS_VARIANT_FOLDED)
  const int fts = elas::fold_table_size(p, q);
  std::vector<double> g(q), w(q), tabh(2 * q * n + 2 * fts + 2 * q);
  elas::host_tables(p, q, nullptr, g.data(), w.data(), tabh.data(), tabh.data() + q * n);
  for (int a = 0; a < q; ++a) {   // Gauss points and sqrt weights (geometry-on-the-fly kernel)
    tabh[elas::tables_gauss_offset(p, q, fts) + a] = g[a];
    tabh[elas::tables_gauss_offset(p, q, fts) + q + a] = std::sqrt(w[a]);
  }
  elas::host_fold_table(p, q, tabh.data(), tabh.data() + 2 * q * n);
  elas::host_fold_table(p, q, tabh.data() + q * n, tabh.data() + 2 * q * n + fts);

  double *dV = nullptr, *dlam = nullptr, *dmu = nullptr;
  int* dbad = nullptr;
  auto cleanup = [&]() {
    cudaFree(dV);
    cudaFree(dlam);
    cudaFree(dmu);
    cudaFree(dbad);
  };
  cudaError_t e;
  const int qlayout = op->variant == ELAS_VARIANT_TENSOR        ? elas::QD_LAYOUT_TC6
                      : op->variant == ELAS_VARIANT_THREAD      ? elas::QD_LAYOUT_E32
                      : op->variant == ELAS_VARIANT_FOLDED_F32 ? elas::QD_LAYOUT_LINES_F32
                      : op->variant == ELAS_VARIANT_FOLDED_OTF ? (p == 1 ? elas::QD_LAYOUT_OTF32 : elas::QD_LAYOUT_OTF)
                                                                : elas::QD_LAYOUT_LINES;
  op->qlayout = qlayout;
  const size_t qbytes = elas::qd_word_bytes(qlayout) * (size_t)elas::qd_stride(q, qlayout) * (size_t)elas::qd_elems(ne, qlayout);
  if ((e = cudaMalloc(&op->qd, qbytes)) != cudaSuccess ||
      (e = cudaMalloc(&op->rr, sizeof(double) * ne)) != cudaSuccess ||
      (e = cudaMalloc(&op->tab, sizeof(double) * tabh.size())) != cudaSuccess ||
      (e = cudaMalloc(&dV, sizeof(double) * V.size())) != cudaSuccess ||
      (e = cudaMalloc(&dlam, sizeof(double) * ne)) != cudaSuccess ||
      (e = cudaMalloc(&dmu, sizeof(double) * ne)) != cudaSuccess ||
      (e = cudaMalloc(&dbad, sizeof(int))) != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "cudaMalloc (operator setup)");
  }
  int rc = ELAS_OK;
  do {
    std::vector<float> tabf(tabh.begin(), tabh.end());
    if ((e = cudaMalloc(&op->tabf, sizeof(float) * tabf.size())) ||
        (e = cudaMemcpy(op->tabf, tabf.data(), sizeof(float) * tabf.size(), cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(op->tab, tabh.data(), sizeof(double) * tabh.size(), cudaMemcpyHostToDevice)) ||
        (e = elas::apply_eo_upload(p, q, tabh.data() + 2 * q * (p + 1))) ||
        (e = cudaMemcpy(dV, V.data(), sizeof(double) * V.size(), cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(dlam, lam.data(), sizeof(double) * ne, cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(dmu, muv.data(), sizeof(double) * ne, cudaMemcpyHostToDevice)) ||
        (e = cudaMemset(dbad, 0, sizeof(int)))) {
      rc = cuda_fail(e, "cudaMemcpy (operator setup)");
      break;
    }
    if ((e = elas::launch_qdata(p, q, qlayout, s, dV, dlam, dmu, g.data(), w.data(), op->qd, op->rr, dbad, op->stream)) ||
        (e = cudaStreamSynchronize(op->stream))) {
      rc = cuda_fail(e, "qdata setup kernel");
      break;
    }
    int bad = 0;
    if ((e = cudaMemcpy(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost))) {
      rc = cuda_fail(e, "cudaMemcpy");
      break;
    }
    if (bad) {
      set_error("det J <= 0 at some quadrature point (inverted or degenerate element)");
      rc = ELAS_EGEOM;
    }
  } while (0);
  cleanup();
  return rc;
}

int range_apply(elas_op* op, const double* x, double* y, int64_t e0, int64_t e1, cudaStream_t st, bool acc = false) {
  if (e1 <= e0) return ELAS_OK;
  Slab sl = op->slab;   // sl.accumulate: the fine-grained kernel's interior nodes take plain stores only when 0
  sl.accumulate = acc ? 1u : 0u;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (op->prof) {
    while (op->prof_ev.size() < op->prof_used + 2) {
      cudaEvent_t ev;
      CUDA_OR(cudaEventCreate(&ev), "cudaEventCreate");
      op->prof_ev.push_back(ev);
    }
    ev0 = op->prof_ev[op->prof_used];
    ev1 = op->prof_ev[op->prof_used + 1];
    op->prof_used += 2;
    CUDA_OR(cudaEventRecord(ev0, st), "cudaEventRecord");
  }
  cudaError_t e;
  if (op->deterministic) {
    // 8 colors in a fixed order over the element layers [e0, e1) (whole layers: e0, e1 are
    // multiples of nx ny); a color's lattice: parity (cx, cy, cz) per axis
    const Slab& s = op->slab;
    const int64_t layer = (int64_t)s.nx * s.ny;
    const int z0 = (int)(e0 / layer), z1 = (int)(e1 / layer);
    e = cudaSuccess;
    for (int c = 0; c < 8 && e == cudaSuccess; ++c) {
      const int cx = c & 1, cy = (c >> 1) & 1, cz = c >> 2;
      const int ncx = (s.nx - cx + 1) / 2, ncy = (s.ny - cy + 1) / 2;
      const int iz0 = (z0 - cz + 1) / 2 > 0 ? (z0 - cz + 1) / 2 : 0;   // first iz with 2 iz + cz >= z0
      const int iz1 = (z1 - cz + 1) / 2 > 0 ? (z1 - cz + 1) / 2 : 0;   // first iz with 2 iz + cz >= z1
      const int64_t cnt = (int64_t)ncx * ncy * (iz1 > iz0 ? iz1 - iz0 : 0);
      if (cnt <= 0) continue;
      const int cm[6] = {cx, cy, cz, ncx, ncy, iz0};
      e = elas::apply_eo_launch(op->p, op->q, op->variant == ELAS_VARIANT_FOLDED_F32, s, x, y, op->qd, op->rr,
                                op->variant == ELAS_VARIANT_FOLDED_F32 ? (const void*)op->tabf : (const void*)op->tab,
                                0, cnt, st, cm, op->variant == ELAS_VARIANT_FOLDED_OTF, op->cc);
    }
  } else if (op->variant >= ELAS_VARIANT_ABL_PA) {
    e = elas::ablation_apply(op, op->variant - ELAS_VARIANT_ABL_PA, x, y, e0, e1, st);
  } else
  e = op->variant == ELAS_VARIANT_TENSOR
                      ? elas::apply_tc_launch(op->slab, x, y, op->qd, op->rr, op->tab, e0, e1, st)
                  : op->variant == ELAS_VARIANT_THREAD
                      ? elas::apply_p1t_launch(op->q, op->slab, x, y, op->qd, op->rr, op->tab, e0, e1, st)
                  : op->variant == ELAS_VARIANT_FOLDED
                      ? elas::apply_eo_launch(op->p, op->q, 0, sl, x, y, op->qd, op->rr, op->tab, e0, e1, st,
                                              nullptr, 0, op->cc)
                  : op->variant == ELAS_VARIANT_FOLDED_F32
                      ? elas::apply_eo_launch(op->p, op->q, 1, op->slab, x, y, op->qd, op->rr, op->tabf, e0, e1, st)
                  : (op->variant == ELAS_VARIANT_FOLDED_OTF && op->p == 1)   // thread-per-element kernel
                      ? elas::apply_p1t_launch(op->q, op->slab, x, y, op->qd, op->rr, op->tab, e0, e1, st, 1)
                  : op->variant == ELAS_VARIANT_FOLDED_OTF
                      ? elas::apply_eo_launch(op->p, op->q, 0, op->slab, x, y, op->qd, op->rr, op->tab, e0, e1, st,
                                              nullptr, 1)
                      : elas::apply_launch(op->p, op->q, op->slab, x, y, op->qd, op->rr, op->tab, e0, e1, st);
  if (e != cudaSuccess) return cuda_fail(e, "apply kernel launch");
  if (op->prof) CUDA_OR(cudaEventRecord(ev1, st), "cudaEventRecord");
  return ELAS_OK;
}

}  // namespace

namespace elas {

int attach_comm(elas_op* op, ncclComm_t comm) {
  if (!op || !comm || op->nranks < 2 || !op->external) {
    set_error("attach_comm: needs an external-mode slab operator and a communicator");
    return ELAS_EINVAL;
  }
  CUDA_OR(cudaStreamCreateWithFlags(&op->comm_stream, cudaStreamNonBlocking), "cudaStreamCreate");
  CUDA_OR(cudaEventCreateWithFlags(&op->ev_boundary, cudaEventDisableTiming), "cudaEventCreate");
  CUDA_OR(cudaEventCreateWithFlags(&op->ev_comm, cudaEventDisableTiming), "cudaEventCreate");
  op->comm = comm;
  op->comm_borrowed = true;
  op->external = false;
  return ELAS_OK;
}

// The interface sum (A6, PAPER.md:169 P^T) in two halves around the interior elements.
// begin: after the boundary layers, the partial interface planes of y leave on the comm stream --
//   NCCL send/recv into the neighbours' halo buffers, or (peer mode, elas_set_peer_exchange) a
//   direct copy into the neighbour's IPC-mapped halo over NVLink followed by a release store of
//   the exchange epoch into the neighbour's flag;
// end: the received halos are added into y (the same plane-add kernel in both modes, so the
//   replicated planes are bitwise equal: a + b on one rank, b + a on the other).  Peer mode first
//   waits on the flag the neighbour set (a one-thread kernel spinning on its own device memory,
//   written by the other GPU), then tells the neighbour its halo may be overwritten again.
int exchange_begin(elas_op* op, double* y) {
  if (op->nranks == 1 || op->external) return ELAS_OK;
  const Slab& s = op->slab;
  cudaStream_t st = op->stream;
  const bool lo = op->rank > 0, hi = op->rank < op->nranks - 1;
  const int64_t plane = (int64_t)s.Nx * s.Ny;
  CUDA_OR(cudaEventRecord(op->ev_boundary, st), "cudaEventRecord");
  CUDA_OR(cudaStreamWaitEvent(op->comm_stream, op->ev_boundary, 0), "cudaStreamWaitEvent");
  if (op->peer_on) {
    const unsigned long long ep = ++op->peer_epoch;
    cudaStream_t cs = op->comm_stream;
    if (lo) {   // my bottom plane -> the lower rank's halo_hi
      CUDA_OR(launch_wait_flag(op->peer_flags + PF_CONSUMED_LO, ep - 1, cs), "peer wait");
      for (int c = 0; c < 3; ++c)
        CUDA_OR(cudaMemcpyAsync(op->peer_lo_halo + c * plane, y + c * s.nodes, sizeof(double) * plane,
                                cudaMemcpyDeviceToDevice, cs), "peer copy");
      CUDA_OR(launch_signal_flag(op->peer_lo_flags + PF_FILLED_HI, ep, cs), "peer signal");
    }
    if (hi) {   // my top plane -> the upper rank's halo_lo
      CUDA_OR(launch_wait_flag(op->peer_flags + PF_CONSUMED_HI, ep - 1, cs), "peer wait");
      for (int c = 0; c < 3; ++c)
        CUDA_OR(cudaMemcpyAsync(op->peer_hi_halo + c * plane, y + c * s.nodes + (int64_t)(s.Nz - 1) * plane,
                                sizeof(double) * plane, cudaMemcpyDeviceToDevice, cs), "peer copy");
      CUDA_OR(launch_signal_flag(op->peer_hi_flags + PF_FILLED_LO, ep, cs), "peer signal");
    }
  } else {
    NCCL_OR(ncclGroupStart(), "ncclGroupStart");
    for (int c = 0; c < 3; ++c) {
      if (lo) {
        NCCL_OR(ncclSend(y + c * s.nodes, plane, ncclDouble, op->rank - 1, op->comm, op->comm_stream), "ncclSend");
        NCCL_OR(ncclRecv(op->halo_lo + c * plane, plane, ncclDouble, op->rank - 1, op->comm, op->comm_stream), "ncclRecv");
      }
      if (hi) {
        NCCL_OR(ncclSend(y + c * s.nodes + (int64_t)(s.Nz - 1) * plane, plane, ncclDouble, op->rank + 1, op->comm,
                         op->comm_stream), "ncclSend");
        NCCL_OR(ncclRecv(op->halo_hi + c * plane, plane, ncclDouble, op->rank + 1, op->comm, op->comm_stream), "ncclRecv");
      }
    }
    NCCL_OR(ncclGroupEnd(), "ncclGroupEnd");
  }
  CUDA_OR(cudaEventRecord(op->ev_comm, op->comm_stream), "cudaEventRecord");
  return ELAS_OK;
}

int exchange_end(elas_op* op, double* y) {
  if (op->nranks == 1 || op->external) return ELAS_OK;
  const Slab& s = op->slab;
  cudaStream_t st = op->stream;
  const bool lo = op->rank > 0, hi = op->rank < op->nranks - 1;
  // my own sends are done with y's boundary planes before anything later on st writes them
  CUDA_OR(cudaStreamWaitEvent(st, op->ev_comm, 0), "cudaStreamWaitEvent");
  const unsigned long long ep = op->peer_epoch;
  if (lo) {
    if (op->peer_on) CUDA_OR(launch_wait_flag(op->peer_flags + PF_FILLED_LO, ep, st), "peer wait");
    CUDA_OR(launch_plane_add(s, 0, y, op->halo_lo, st), "plane add launch");
    if (op->peer_on) CUDA_OR(launch_signal_flag(op->peer_lo_flags + PF_CONSUMED_HI, ep, st), "peer signal");
  }
  if (hi) {
    if (op->peer_on) CUDA_OR(launch_wait_flag(op->peer_flags + PF_FILLED_HI, ep, st), "peer wait");
    CUDA_OR(launch_plane_add(s, s.Nz - 1, y, op->halo_hi, st), "plane add launch");
    if (op->peer_on) CUDA_OR(launch_signal_flag(op->peer_hi_flags + PF_CONSUMED_LO, ep, st), "peer signal");
  }
  return ELAS_OK;
}

int exchange_planes(elas_op* op, double* y) {
  int rc = exchange_begin(op, y);
  return rc ? rc : exchange_end(op, y);
}

}  // namespace elas

extern "C" {

int elas_version(void) { return ELAS_VERSION; }

int elas_debug_checks(int* first_line, int selftest) {
  unsigned count = 0, line = 0;
  if (selftest) {
    CUDA_OR(elas::launch_dcheck_selftest(nullptr), "debug self-test launch");
    CUDA_OR(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  }
  cudaError_t (*readers[])(unsigned*, unsigned*) = {
      elas::dcheck_setup, elas::dcheck_p1t, elas::dcheck_tc,
      elas::dcheck_eo_p1, elas::dcheck_eo_p2, elas::dcheck_eo_p3, elas::dcheck_eo_p4,
      elas::dcheck_eo_p5, elas::dcheck_eo_p6, elas::dcheck_eo_p7, elas::dcheck_eo_p8,
      elas::dcheck_simt_p1, elas::dcheck_simt_p2, elas::dcheck_simt_p3, elas::dcheck_simt_p4,
      elas::dcheck_simt_p5, elas::dcheck_simt_p6, elas::dcheck_simt_p7, elas::dcheck_simt_p8};
  for (auto rd : readers) CUDA_OR(rd(&count, &line), "debug check read");
  if (first_line) *first_line = (int)line;
  return (int)count;
}

int elas_debug_build(void) { return ELAS_DEBUG; }

int elas_set_peer_exchange(elas_op* op, int on) {
  if (!op) { set_error("elas_set_peer_exchange: NULL op"); return ELAS_EINVAL; }
  if (op->nranks < 2 || op->external || !op->comm) {
    set_error("elas_set_peer_exchange: needs an NCCL-mode slab operator (nranks > 1, nccl_id given)");
    return ELAS_EINVAL;
  }
  if (!on) { op->peer_on = false; return ELAS_OK; }
  if (op->peer_flags) { op->peer_on = true; return ELAS_OK; }
  const bool lo = op->rank > 0, hi = op->rank < op->nranks - 1;
  CUDA_OR(cudaStreamSynchronize(op->stream), "cudaStreamSynchronize");
  CUDA_OR(cudaStreamSynchronize(op->comm_stream), "cudaStreamSynchronize");
  CUDA_OR(cudaMalloc(&op->peer_flags, sizeof(unsigned long long) * elas::PF_COUNT), "cudaMalloc (peer flags)");
  CUDA_OR(cudaMemset(op->peer_flags, 0, sizeof(unsigned long long) * elas::PF_COUNT), "cudaMemset (peer flags)");
  // my IPC handles: halo_lo, halo_hi, flags -> both neighbours (NCCL send/recv of the bytes; the
  // exchange also orders every rank's zeroed flags before any neighbour can signal them)
  cudaIpcMemHandle_t mine[3], from_lo[3], from_hi[3];
  CUDA_OR(cudaIpcGetMemHandle(&mine[0], op->halo_lo), "cudaIpcGetMemHandle");
  CUDA_OR(cudaIpcGetMemHandle(&mine[1], op->halo_hi), "cudaIpcGetMemHandle");
  CUDA_OR(cudaIpcGetMemHandle(&mine[2], op->peer_flags), "cudaIpcGetMemHandle");
  const size_t hb = sizeof(mine);
  char* dbuf = nullptr;
  CUDA_OR(cudaMalloc(&dbuf, 3 * hb), "cudaMalloc (handle exchange)");
  CUDA_OR(cudaMemcpy(dbuf, mine, hb, cudaMemcpyHostToDevice), "cudaMemcpy");
  ncclResult_t nr = ncclGroupStart();
  if (nr == ncclSuccess && lo) {
    nr = ncclSend(dbuf, hb, ncclInt8, op->rank - 1, op->comm, op->comm_stream);
    if (nr == ncclSuccess) nr = ncclRecv(dbuf + hb, hb, ncclInt8, op->rank - 1, op->comm, op->comm_stream);
  }
  if (nr == ncclSuccess && hi) {
    nr = ncclSend(dbuf, hb, ncclInt8, op->rank + 1, op->comm, op->comm_stream);
    if (nr == ncclSuccess) nr = ncclRecv(dbuf + 2 * hb, hb, ncclInt8, op->rank + 1, op->comm, op->comm_stream);
  }
  ncclResult_t ne = ncclGroupEnd();
  cudaError_t ce = cudaStreamSynchronize(op->comm_stream);
  if (ce == cudaSuccess) ce = cudaMemcpy(from_lo, dbuf + hb, hb, cudaMemcpyDeviceToHost);
  if (ce == cudaSuccess) ce = cudaMemcpy(from_hi, dbuf + 2 * hb, hb, cudaMemcpyDeviceToHost);
  cudaFree(dbuf);
  if (nr != ncclSuccess) return nccl_fail(nr, "handle exchange");
  if (ne != ncclSuccess) return nccl_fail(ne, "handle exchange");
  if (ce != cudaSuccess) return cuda_fail(ce, "handle exchange");
  void* ptr = nullptr;
  if (lo) {   // the lower rank's halo_hi (my bottom plane goes there) and its flags
    CUDA_OR(cudaIpcOpenMemHandle(&ptr, from_lo[1], cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    op->peer_lo_halo = static_cast<double*>(ptr);
    CUDA_OR(cudaIpcOpenMemHandle(&ptr, from_lo[2], cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    op->peer_lo_flags = static_cast<unsigned long long*>(ptr);
  }
  if (hi) {   // the upper rank's halo_lo and its flags
    CUDA_OR(cudaIpcOpenMemHandle(&ptr, from_hi[0], cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    op->peer_hi_halo = static_cast<double*>(ptr);
    CUDA_OR(cudaIpcOpenMemHandle(&ptr, from_hi[2], cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    op->peer_hi_flags = static_cast<unsigned long long*>(ptr);
  }
  op->peer_epoch = 0;
  op->peer_on = true;
  return ELAS_OK;
}

int elas_nccl_unique_id(void* id_out) {
  if (!id_out) { set_error("elas_nccl_unique_id: NULL output"); return ELAS_EINVAL; }
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id_out, &id, sizeof(id));
  return ELAS_OK;
}

const char* elas_last_error(void) { return elas::g_err.c_str(); }

int elas_slab_range(int32_t nz, int32_t rank, int32_t nranks, int32_t* ez_begin, int32_t* ez_end) {
  if (nranks < 1 || rank < 0 || rank >= nranks || nz < nranks) {
    set_error("elas_slab_range: need 1 <= nranks <= nz and 0 <= rank < nranks");
    return ELAS_EINVAL;
  }
  if (ez_begin) *ez_begin = (int32_t)(((int64_t)rank * nz) / nranks);
  if (ez_end) *ez_end = (int32_t)(((int64_t)(rank + 1) * nz) / nranks);
  return ELAS_OK;
}

int elas_tables(int p, int q, double* nodes, double* points, double* weights, double* B, double* D) {
  int rc = elas::host_tables(p, q, nodes, points, weights, B, D);
  if (rc) set_error("elas_tables: need 1 <= p <= 8 and 1 <= q <= 16");
  return rc;
}

elas_op* elas_create(const elas_mesh* m, int p, int q, const double* lambda, const double* mu) {
  return elas_create_ex(m, p, q, lambda, mu, ELAS_VARIANT_AUTO);
}

elas_op* elas_create_ex(const elas_mesh* m, int p, int q, const double* lambda, const double* mu, int variant) {
  elas::g_err.clear();
  if (variant < ELAS_VARIANT_AUTO || variant > ELAS_VARIANT_ABL_VOIGT) {
    set_error("elas_create_ex: unknown variant");
    return nullptr;
  }
  const bool tc_ok = (p == 6 && q == 8);
  const bool thread_ok = (p == 1);
  if (variant == ELAS_VARIANT_TENSOR && !tc_ok) {
    set_error("elas_create_ex: the tensor-core variant exists for p = 6, q = 8 only");
    return nullptr;
  }
  if (variant == ELAS_VARIANT_THREAD && !thread_ok) {
    set_error("elas_create_ex: the one-thread-per-element variant exists for p = 1 only");
    return nullptr;
  }
  if (!m || !lambda || !mu) { set_error("elas_create: NULL mesh/lambda/mu"); return nullptr; }
  if (p < 1 || p > 8) { set_error("elas_create: p must be in [1, 8]"); return nullptr; }
  if (q != p + 1 && q != p + 2) { set_error("elas_create: q must be p+1 or p+2"); return nullptr; }
  if (m->nx < 1 || m->ny < 1 || m->nz < 1) { set_error("elas_create: nx, ny, nz must be >= 1"); return nullptr; }
  if (!m->vertices && !(m->lx > 0 && m->ly > 0 && m->lz > 0)) {
    set_error("elas_create: lx, ly, lz must be > 0 when vertices == NULL");
    return nullptr;
  }
  if (m->dirichlet_faces & ~63u) { set_error("elas_create: unknown Dirichlet face bits"); return nullptr; }
  const int64_t Nx = (int64_t)m->nx * p + 1, Ny = (int64_t)m->ny * p + 1;
  if (Nx * Ny * ((int64_t)m->nz * p + 1) * 3 >= (int64_t)1 << 31) {
    // 32-bit node indices inside the kernels (I, J, K); vector offsets are 64-bit but we
    // keep the global dof count below 2^31 as documented.
    set_error("elas_create: more than 2^31 - 1 dofs per rank is not supported");
    return nullptr;
  }
  elas_op* op = new elas_op();
  op->p = p;
  op->q = q;
  if (variant == ELAS_VARIANT_AUTO)
    variant = (tc_ok && kAutoTensor)       ? ELAS_VARIANT_TENSOR
              : (thread_ok && kAutoThread) ? ELAS_VARIANT_THREAD
              : kAutoFolded                ? ELAS_VARIANT_FOLDED
                                           : ELAS_VARIANT_SIMT;
  op->variant = variant;
  op->nranks = m->nranks < 1 ? 1 : m->nranks;
  op->rank = m->rank;
  int32_t b, e;
  if (elas_slab_range(m->nz, op->rank, op->nranks, &b, &e) != ELAS_OK) { free_op(op); return nullptr; }
  op->ez0 = b;
  op->ez1 = e;
  op->nz_global = m->nz;
  cudaGetDevice(&op->device);
  int rc = build(op, m, lambda, mu);
  if (rc != ELAS_OK) { free_op(op); return nullptr; }
  if (op->nranks > 1) {
    const size_t pbytes = sizeof(double) * 3 * (size_t)op->slab.Nx * op->slab.Ny;
    cudaError_t ce;
    if ((ce = cudaMalloc(&op->halo_lo, pbytes)) || (ce = cudaMalloc(&op->halo_hi, pbytes))) {
      cuda_fail(ce, "cudaMalloc (halo planes)");
      free_op(op);
      return nullptr;
    }
    if (m->nccl_id) {
      ncclUniqueId id;
      std::memcpy(&id, m->nccl_id, sizeof(id));
      ncclResult_t r = ncclCommInitRank(&op->comm, op->nranks, id, op->rank);
      if (r != ncclSuccess) { nccl_fail(r, "ncclCommInitRank"); op->comm = nullptr; free_op(op); return nullptr; }
      if ((ce = cudaStreamCreateWithFlags(&op->comm_stream, cudaStreamNonBlocking)) ||
          (ce = cudaEventCreateWithFlags(&op->ev_boundary, cudaEventDisableTiming)) ||
          (ce = cudaEventCreateWithFlags(&op->ev_comm, cudaEventDisableTiming))) {
        cuda_fail(ce, "stream/event creation");
        free_op(op);
        return nullptr;
      }
    } else {
      op->external = true;
    }
  }
  return op;
}

elas_op* elas_create_aniso(const elas_mesh* m, int p, int q, const double* C21) {
  elas::g_err.clear();
  if (!m || !C21) { set_error("elas_create_aniso: NULL mesh/C"); return nullptr; }
  const int64_t nc = 21 * (m->material_per_element ? (int64_t)m->nx * m->ny * m->nz : 1);
  for (int64_t i = 0; i < nc; ++i)
    if (!std::isfinite(C21[i])) { set_error("elas_create_aniso: non-finite Voigt matrix entry"); return nullptr; }
  // quadrature data A~ = sqrt(W) J^{-1}: the isotropic setup with mu = 1, lambda = 0 (r = 0)
  elas_mesh m1 = *m;
  m1.material_per_element = 0;
  const double lam0 = 0.0, mu1 = 1.0;
  elas_op* op = elas_create_ex(&m1, p, q, &lam0, &mu1, ELAS_VARIANT_FOLDED);
  if (!op) return nullptr;
  const int64_t ne = (int64_t)op->slab.nx * op->slab.ny * op->slab.nz;
  const int64_t off = (int64_t)op->ez0 * m->nx * m->ny;
  std::vector<double> cch((size_t)ne * 21);
  for (int64_t e = 0; e < ne; ++e)
    for (int w = 0; w < 21; ++w) cch[(size_t)e * 21 + w] = m->material_per_element ? C21[(off + e) * 21 + w] : C21[w];
  cudaError_t ce = cudaMalloc(&op->cc, sizeof(double) * cch.size());
  if (!ce) ce = cudaMemcpy(op->cc, cch.data(), sizeof(double) * cch.size(), cudaMemcpyHostToDevice);
  if (ce) { cuda_fail(ce, "cudaMalloc/cudaMemcpy (Voigt matrices)"); free_op(op); return nullptr; }
  return op;
}

void elas_destroy(elas_op* op) {
  if (op) cudaStreamSynchronize(op->stream);
  free_op(op);
}

int64_t elas_local_dofs(const elas_op* op) { return op ? 3 * op->slab.nodes : -1; }

int elas_local_zrange(const elas_op* op, int32_t* ez_begin, int32_t* ez_end) {
  if (!op) { set_error("elas_local_zrange: NULL op"); return ELAS_EINVAL; }
  if (ez_begin) *ez_begin = op->ez0;
  if (ez_end) *ez_end = op->ez1;
  return ELAS_OK;
}

int elas_set_stream(elas_op* op, void* st) {
  if (!op) { set_error("elas_set_stream: NULL op"); return ELAS_EINVAL; }
  op->stream = (cudaStream_t)st;
  return ELAS_OK;
}

int elas_profile(elas_op* op, int enable) {
  if (!op) { set_error("elas_profile: NULL op"); return ELAS_EINVAL; }
  if (enable && !op->prof) op->prof_used = 0;   // enabling starts a fresh window
  op->prof = enable != 0;                          // disabling keeps it for elas_profile_read
  return ELAS_OK;
}

int elas_profile_read(elas_op* op, double* ms, int64_t* launches) {
  if (!op) { set_error("elas_profile_read: NULL op"); return ELAS_EINVAL; }
  double total = 0.0;
  if (op->prof_used) CUDA_OR(cudaEventSynchronize(op->prof_ev[op->prof_used - 1]), "cudaEventSynchronize");
  for (size_t i = 0; i + 1 < op->prof_used; i += 2) {
    float t = 0.f;
    CUDA_OR(cudaEventElapsedTime(&t, op->prof_ev[i], op->prof_ev[i + 1]), "cudaEventElapsedTime");
    total += t;
  }
  if (ms) *ms = total;
  if (launches) *launches = (int64_t)(op->prof_used / 2);
  op->prof_used = 0;
  return ELAS_OK;
}

int elas_variant(const elas_op* op) { return op ? op->variant : -1; }

int elas_set_deterministic(elas_op* op, int on) {
  if (!op) { set_error("elas_set_deterministic: NULL op"); return ELAS_EINVAL; }
  if (on && op->variant != ELAS_VARIANT_FOLDED && op->variant != ELAS_VARIANT_FOLDED_F32 &&
      op->variant != ELAS_VARIANT_FOLDED_OTF) {
    set_error("elas_set_deterministic: the colored scatter exists for the folded variants only");
    return ELAS_EINVAL;
  }
  op->deterministic = on != 0;
  return ELAS_OK;
}

// kernels of ONE element range [z0, z1) of layers: 1, or the non-empty colors in colored mode
static int range_launches(const elas_op* op, int z0, int z1) {
  if (z1 <= z0) return 0;
  if (op->variant >= ELAS_VARIANT_ABL_PA) return 5;   // gather, gradient, pointwise, transpose, scatter
  if (!op->deterministic) return 1;
  const Slab& s = op->slab;
  int n = 0;
  for (int c = 0; c < 8; ++c) {
    const int cx = c & 1, cy = (c >> 1) & 1, cz = c >> 2;
    const int ncx = (s.nx - cx + 1) / 2, ncy = (s.ny - cy + 1) / 2;
    const int iz0 = (z0 - cz + 1) / 2 > 0 ? (z0 - cz + 1) / 2 : 0;
    const int iz1 = (z1 - cz + 1) / 2 > 0 ? (z1 - cz + 1) / 2 : 0;
    if ((int64_t)ncx * ncy * (iz1 > iz0 ? iz1 - iz0 : 0) > 0) ++n;
  }
  return n;
}

int elas_launches_per_apply(const elas_op* op) {
  if (!op) return -1;
  // init = a memset (not a kernel) + the Dirichlet-face copy kernel when faces are constrained
  int n = op->slab.faces ? 1 : 0;
  const int nzl = op->ez1 - op->ez0;
  if (op->nranks == 1 || op->external) return n + range_launches(op, 0, nzl);
  const bool lo = op->rank > 0, hi = op->rank < op->nranks - 1;
  int i0 = 0, i1 = nzl;
  if (lo) { n += range_launches(op, 0, 1); i0 = 1; }
  if (hi && nzl - 1 >= i0) { n += range_launches(op, nzl - 1, nzl); i1 = nzl - 1; }
  else if (hi) i1 = i0;
  n += range_launches(op, i0, i1);             // interior
  n += (int)lo + (int)hi;                      // plane adds
  return n;
}

int elas_apply(elas_op* op, const double* x, double* y) {
  if (!op || !x || !y) { set_error("elas_apply: NULL argument"); return ELAS_EINVAL; }
  if (x == y) { set_error("elas_apply: x and y must not alias"); return ELAS_EINVAL; }
  if (((uintptr_t)x | (uintptr_t)y) & 7u) { set_error("elas_apply: x, y must be 8-byte aligned"); return ELAS_EINVAL; }
  const Slab& s = op->slab;
  cudaStream_t st = op->stream;
  CUDA_OR(elas::launch_init(s, x, y, st), "init kernel launch");
  const int64_t layer = (int64_t)s.nx * s.ny;
  const int64_t ne = layer * s.nz;
  if (op->nranks == 1 || op->external) return range_apply(op, x, y, 0, ne, st);

  // NCCL slab mode: boundary layers, exchange overlapped with the interior, plane add.
  const bool lo = op->rank > 0, hi = op->rank < op->nranks - 1;
  int64_t int0 = 0, int1 = ne;
  int rc;
  if (lo) { if ((rc = range_apply(op, x, y, 0, layer, st))) return rc; int0 = layer; }
  if (hi && ne - layer >= int0) { if ((rc = range_apply(op, x, y, ne - layer, ne, st))) return rc; int1 = ne - layer; }
  else if (hi) int1 = int0;
  if ((rc = elas::exchange_begin(op, y))) return rc;     // overlapped with the interior elements
  if ((rc = range_apply(op, x, y, int0, int1, st))) return rc;
  return elas::exchange_end(op, y);
}

int elas_apply_add(elas_op* op, const double* x, double* y) {
  if (!op || !x || !y) { set_error("elas_apply_add: NULL argument"); return ELAS_EINVAL; }
  if (x == y) { set_error("elas_apply_add: x and y must not alias"); return ELAS_EINVAL; }
  if (((uintptr_t)x | (uintptr_t)y) & 7u) { set_error("elas_apply_add: x, y must be 8-byte aligned"); return ELAS_EINVAL; }
  if (op->nranks != 1) {
    set_error("elas_apply_add: single-GPU operators only (the interface sum needs the partial planes alone)");
    return ELAS_EINVAL;
  }
  const Slab& s = op->slab;
  CUDA_OR(elas::launch_face_add(s, x, y, op->stream), "face add launch");
  return range_apply(op, x, y, 0, (int64_t)s.nx * s.ny * s.nz, op->stream, true);
}

int elas_interface_add(elas_op* op, double* y, const double* lo_halo, const double* hi_halo) {
  if (!op || !y) { set_error("elas_interface_add: NULL argument"); return ELAS_EINVAL; }
  if (!op->external) { set_error("elas_interface_add: only for external-exchange ops (nranks > 1, nccl_id NULL)"); return ELAS_EINVAL; }
  const bool lo = op->rank > 0, hi = op->rank < op->nranks - 1;
  if ((lo_halo != nullptr) != lo || (hi_halo != nullptr) != hi) {
    set_error("elas_interface_add: halo pointers do not match the rank's neighbours");
    return ELAS_EINVAL;
  }
  if (lo) CUDA_OR(elas::launch_plane_add(op->slab, 0, y, lo_halo, op->stream), "plane add launch");
  if (hi) CUDA_OR(elas::launch_plane_add(op->slab, op->slab.Nz - 1, y, hi_halo, op->stream), "plane add launch");
  return ELAS_OK;
}

int elas_apply_host(elas_op* op, const double* xh, double* yh) {
  if (!op || !xh || !yh) { set_error("elas_apply_host: NULL argument"); return ELAS_EINVAL; }
  const size_t bytes = sizeof(double) * 3 * (size_t)op->slab.nodes;
  if (!op->xs) CUDA_OR(cudaMalloc(&op->xs, bytes), "cudaMalloc (staging)");
  if (!op->ys) CUDA_OR(cudaMalloc(&op->ys, bytes), "cudaMalloc (staging)");
  const Slab& s = op->slab;
  if (op->nranks > 1 || s.nz < 2) {   // one shot: H2D, apply, D2H
    CUDA_OR(cudaMemcpyAsync(op->xs, xh, bytes, cudaMemcpyHostToDevice, op->stream), "cudaMemcpyAsync H2D");
    int rc = elas_apply(op, op->xs, op->ys);
    if (rc) return rc;
    CUDA_OR(cudaMemcpyAsync(yh, op->ys, bytes, cudaMemcpyDeviceToHost, op->stream), "cudaMemcpyAsync D2H");
    CUDA_OR(cudaStreamSynchronize(op->stream), "cudaStreamSynchronize");
    return ELAS_OK;
  }
  // Pipelined over z-chunks of element layers: the H2D copy of chunk k+1's node planes, the
  // apply of chunk k and the D2H copy of chunk k-1's finished planes run concurrently on three
  // streams (PCIe is full duplex; the apply is ~10x faster than either copy).  Plane K of y is
  // final once every element layer touching it has been applied: after chunk k, planes below
  // its top plane are final.
  const int nchunk = s.nz < ELAS_HOST_CHUNKS ? s.nz : ELAS_HOST_CHUNKS;   // fill + drain ~2/nchunk of the copies
  if (!op->h2d) CUDA_OR(cudaStreamCreateWithFlags(&op->h2d, cudaStreamNonBlocking), "cudaStreamCreate");
  if (!op->d2h) CUDA_OR(cudaStreamCreateWithFlags(&op->d2h, cudaStreamNonBlocking), "cudaStreamCreate");
  while ((int)op->host_ev.size() < 2 * nchunk + 1) {
    cudaEvent_t ev;
    CUDA_OR(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
    op->host_ev.push_back(ev);
  }
  const int64_t plane = (int64_t)s.Nx * s.Ny;
  const int64_t layer = (int64_t)s.nx * s.ny;
  const int p = op->p;
  cudaStream_t st = op->stream;
  // copies must not start before work already queued on the op's stream (e.g. earlier reads of xs)
  CUDA_OR(cudaEventRecord(op->host_ev[2 * nchunk], st), "cudaEventRecord");
  CUDA_OR(cudaStreamWaitEvent(op->h2d, op->host_ev[2 * nchunk], 0), "cudaStreamWaitEvent");
  CUDA_OR(cudaStreamWaitEvent(op->d2h, op->host_ev[2 * nchunk], 0), "cudaStreamWaitEvent");
  auto copy_planes = [&](double* dst, const double* src, int K0, int K1, cudaMemcpyKind kind, cudaStream_t cs) -> int {
    if (K1 <= K0) return ELAS_OK;
    for (int c = 0; c < 3; ++c) {
      const int64_t off = c * s.nodes + (int64_t)K0 * plane;
      CUDA_OR(cudaMemcpyAsync(dst + off, src + off, sizeof(double) * (size_t)(K1 - K0) * plane, kind, cs),
              "cudaMemcpyAsync (chunk)");
    }
    return ELAS_OK;
  };
  int x_done = 0, y_done = 0, rc;   // planes [0, x_done) copied in, [0, y_done) copied out
  for (int k = 0; k < nchunk; ++k) {
    const int z0 = (int)(((int64_t)k * s.nz) / nchunk), z1 = (int)(((int64_t)(k + 1) * s.nz) / nchunk);
    const int top = z1 * p + 1;            // x planes [0, top) needed by layers < z1
    if ((rc = copy_planes(op->xs, xh, x_done, top, cudaMemcpyHostToDevice, op->h2d))) return rc;
    CUDA_OR(cudaEventRecord(op->host_ev[2 * k], op->h2d), "cudaEventRecord");
    CUDA_OR(cudaStreamWaitEvent(st, op->host_ev[2 * k], 0), "cudaStreamWaitEvent");
    CUDA_OR(elas::launch_init_planes(s, x_done, top, op->xs, op->ys, st), "init kernel launch");
    x_done = top;
    if ((rc = range_apply(op, op->xs, op->ys, (int64_t)z0 * layer, (int64_t)z1 * layer, st))) return rc;
    CUDA_OR(cudaEventRecord(op->host_ev[2 * k + 1], st), "cudaEventRecord");
    CUDA_OR(cudaStreamWaitEvent(op->d2h, op->host_ev[2 * k + 1], 0), "cudaStreamWaitEvent");
    const int fin = (k == nchunk - 1) ? s.Nz : z1 * p;   // the top plane waits for the next chunk
    if ((rc = copy_planes(yh, op->ys, y_done, fin, cudaMemcpyDeviceToHost, op->d2h))) return rc;
    y_done = fin;
  }
  CUDA_OR(cudaStreamSynchronize(op->d2h), "cudaStreamSynchronize");
  CUDA_OR(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  return ELAS_OK;
}

}  // extern "C"
