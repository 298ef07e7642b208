// Internal declarations shared by the libelas translation units.
#pragma once
#include <cstdint>
#include <mutex>
#include <string>

#include <cuda_runtime.h>

#include "../../include/elas.h"

// Debug build (ELAS_DEBUG=1, lib/libelas_debug.so): device-side bounds checks on every global
// gather/scatter/quadrature-data index of the apply kernels -- the substitute for
// compute-sanitizer, which is closed on this pool.  A failed check does not trap (a trapped
// kernel can take the GPU down): it counts itself and records its source line in a per-TU
// device word that elas_debug_checks() reads and resets.  In the release build the checks
// compile to nothing.
#ifndef ELAS_DEBUG
#define ELAS_DEBUG 0
#endif
#if defined(__CUDACC__)
namespace elas {
namespace {
__device__ unsigned int g_dcheck[2];   // [0] failed checks, [1] source line of the first failure
}  // namespace
}  // namespace elas
#if ELAS_DEBUG
#define ELAS_DCHECK(cond)                                                                \
  do {                                                                                   \
    if (!(cond)) {                                                                       \
      if (atomicAdd(&::elas::g_dcheck[0], 1u) == 0u) ::elas::g_dcheck[1] = __LINE__;     \
    }                                                                                    \
  } while (0)
#else
#define ELAS_DCHECK(cond) \
  do {                    \
  } while (0)
#endif
// host reader of this translation unit's check words: adds the count, keeps the first line, resets
#define ELAS_DCHECK_READER(NAME)                                                           \
  namespace elas {                                                                         \
  cudaError_t NAME(unsigned* count, unsigned* line) {                                      \
    unsigned h[2] = {0, 0}, z[2] = {0, 0};                                                 \
    cudaError_t e = cudaMemcpyFromSymbol(h, g_dcheck, sizeof(h));                          \
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_dcheck, z, sizeof(z));                  \
    if (h[0] && !*count) *line = h[1];                                                     \
    *count += h[0];                                                                        \
    return e;                                                                              \
  }                                                                                        \
  }
#endif

namespace elas {

// Everything a kernel needs to address one rank's slab (all LOCAL indices).
struct Slab {
  int32_t nx, ny, nz;        // elements per axis (nz = local layers)
  int32_t Nx, Ny, Nz;        // nodes per axis (Nz = nz p + 1)
  int64_t nodes;             // Nx * Ny * Nz
  uint32_t faces;            // Dirichlet face bits, z faces already restricted to this slab
  uint32_t accumulate;       // 1: y += A x (elas_apply_add): no plain stores of element-interior nodes
};

// Launch configuration the host needs for one (p, q) kernel instance.
struct ApplyLaunch {
  int threads;               // CTA size
  int elems_per_cta;         // EB
  size_t smem_bytes;         // dynamic shared memory
};

// Host tables (elas_tables.cpp): GLL nodes, Gauss-Legendre rule, barycentric Lagrange.
int host_tables(int p, int q, double* nodes, double* points, double* weights, double* B, double* D);
// Even-odd folded copy of one table (elas_tables.cpp); op tables = B | D | fold(B) | fold(D).
int fold_table_size(int p, int q);
void host_fold_table(int p, int q, const double* T, double* out);
// GMG 1D prolongation from a coarse element to its two children, (2p+1) x (p+1) (elas_tables.cpp)
int host_prolongation_1d(int p, double* M);

// folded-SIMT variant (elas_apply_eo_p<P>.cu); fp32 != 0: the mixed-precision instance (FP32
// qdata, tables and arithmetic; FP64 x, y and scatter)
cudaError_t apply_eo_info(int p, int q, int fp32, ApplyLaunch* info);
// color == nullptr: elements [e_begin, e_end) with atomic scatter.  color = {cx, cy, cz, ncx, ncy,
// iz0}: the linear range [e_begin, e_end) of one color's element lattice, plain-RMW scatter.
// otf = 1: geometry on the fly (FP64 only; qd = geo[e][GEO_WORDS], QD_LAYOUT_OTF)
// cc != nullptr: anisotropic material (21 Voigt words per element; FP64 only)
// folded tables (2 * fold_table_size doubles) into the folded kernels' constant bank (ELAS_EO_CTAB)
cudaError_t apply_eo_upload(int p, int q, const double* fold);
cudaError_t apply_eo_launch(int p, int q, int fp32, const Slab& s, const double* x, double* y, const void* qd,
                            const double* rr, const void* tables, int64_t e_begin, int64_t e_end,
                            cudaStream_t st, const int* color = nullptr, int otf = 0, const double* cc = nullptr);

// Per-degree translation units (elas_apply_p<P>.cu) export these; q must be p+1 or p+2.
// Returns cudaSuccess or an error; `info` only queries the configuration.
cudaError_t apply_info(int p, int q, ApplyLaunch* info);
cudaError_t apply_launch(int p, int q, const Slab& s, const double* x, double* y, const double* qd,
                         const double* rr, const double* tables, int64_t e_begin, int64_t e_end,
                         cudaStream_t st);

// FP64 tensor-core variant (elas_apply_tc.cu), p = 6, q = 8 only.
cudaError_t apply_tc_info(ApplyLaunch* info);
cudaError_t apply_tc_launch(const Slab& s, const double* x, double* y, const double* qd, const double* rr,
                            const double* tables, int64_t e_begin, int64_t e_end, cudaStream_t st);

// qdata layouts: 0 = qd[e][a1][f][a3 + q a2] (SIMT kernel), 1 = fragment order of the tensor-core
// kernel: qd[e][slice a1/2][r][f][lane], r = 2 (a1 % 2) + a3 % 2, lane = 4 a2 + a3 / 2.
// 2 = lane-interleaved blocks of 32 elements for the one-thread-per-element p = 1 kernel:
//     qd[e / 32][pt][f][e % 32], pt = a1 + q (a2 + q a3).
// 3 = layout 0 in FP32 words (mixed-precision folded kernel), element stride rounded to 4 floats.
// 4 = geometry on the fly (ELAS_VARIANT_FOLDED_OTF): per element only the trilinear map's
//     Jacobian coefficients, geo[e][GEO_WORDS]: dx/dxi1 = c0 + c1 xi2 + c2 xi3 + c3 xi2 xi3,
//     dx/dxi2 = e0 + e1 xi1 + e2 xi3 + e3 xi1 xi3, dx/dxi3 = f0 + f1 xi1 + f2 xi2 + f3 xi1 xi2
//     (3-vectors: c0..c3 at 0..11, e at 12..23, f at 24..35), sqrt(mu_e) at 36.
// 5 = layout 4 lane-interleaved over blocks of 32 elements (p = 1 thread-per-element kernel):
//     geo32[e / 32][w][e % 32].
enum { QD_LAYOUT_LINES = 0, QD_LAYOUT_TC6 = 1, QD_LAYOUT_E32 = 2, QD_LAYOUT_LINES_F32 = 3, QD_LAYOUT_OTF = 4,
       QD_LAYOUT_OTF32 = 5 };
constexpr int GEO_WORDS = 40;

// qdata doubles per element: 9 q^3 rounded up to even so every element starts 16-B aligned
// (TMA bulk copies need 16-B aligned addresses and sizes).
constexpr int qd_stride_lines(int q) { return (9 * q * q * q + 1) & ~1; }
inline int qd_stride(int q, int layout) {
  return layout == QD_LAYOUT_LINES       ? qd_stride_lines(q)
         : layout == QD_LAYOUT_LINES_F32 ? (9 * q * q * q + 3) & ~3
         : (layout == QD_LAYOUT_OTF || layout == QD_LAYOUT_OTF32) ? GEO_WORDS
                                         : 9 * q * q * q;
}
// op tables: B | D | fold(B) | fold(D) | Gauss points g[q] | sqrt(w)[q]
inline int tables_gauss_offset(int p, int q, int fts) { return 2 * q * (p + 1) + 2 * fts; }
inline size_t qd_word_bytes(int layout) { return layout == QD_LAYOUT_LINES_F32 ? 4 : 8; }
// elements the qdata allocation must cover (E32 pads to whole blocks of 32)
inline int64_t qd_elems(int64_t ne, int layout) {
  return (layout == QD_LAYOUT_E32 || layout == QD_LAYOUT_OTF32) ? (ne + 31) / 32 * 32 : ne;
}

// one-thread-per-element kernel, p = 1 (elas_apply_p1t.cu)
// otf = 1: geometry on the fly (qd = geo32, QD_LAYOUT_OTF32; tables must carry the Gauss points)
cudaError_t apply_p1t_launch(int q, const Slab& s, const double* x, double* y, const double* qd, const double* rr,
                             const double* tables, int64_t e_begin, int64_t e_end, cudaStream_t st, int otf = 0);

// Kernels in elas_setup.cu
cudaError_t launch_qdata(int p, int q, int layout, const Slab& s, const double* verts, const double* lam,
                         const double* mu, const double* gpts, const double* gw, double* qd,
                         double* rr, int* bad, cudaStream_t st);
cudaError_t launch_init(const Slab& s, const double* x, double* y, cudaStream_t st);
cudaError_t launch_init_planes(const Slab& s, int K0, int K1, const double* x, double* y, cudaStream_t st);
// y += x on the constrained dofs (each once): the identity rows of the accumulating apply
// y = x on every constrained row (whole slab)
cudaError_t launch_face_copy(const Slab& s, const double* x, double* y, cudaStream_t st);
cudaError_t launch_face_add(const Slab& s, const double* x, double* y, cudaStream_t st);
cudaError_t launch_plane_add(const Slab& s, int which_plane, double* y, const double* halo,
                             cudaStream_t st);
// peer-mode interface exchange: one thread spins (acquire, system scope) until *flag >= target;
// one thread stores value into a (possibly peer, IPC-mapped) flag with release semantics
cudaError_t launch_wait_flag(const unsigned long long* flag, unsigned long long target, cudaStream_t st);
cudaError_t launch_signal_flag(unsigned long long* flag, unsigned long long value, cudaStream_t st);
// debug build: the per-translation-unit readers of the device check words (ELAS_DCHECK_READER)
cudaError_t launch_dcheck_selftest(cudaStream_t st);
#define ELAS_DCHECK_DECL(NAME) cudaError_t NAME(unsigned* count, unsigned* line);
ELAS_DCHECK_DECL(dcheck_setup) ELAS_DCHECK_DECL(dcheck_p1t) ELAS_DCHECK_DECL(dcheck_tc)
ELAS_DCHECK_DECL(dcheck_eo_p1) ELAS_DCHECK_DECL(dcheck_eo_p2) ELAS_DCHECK_DECL(dcheck_eo_p3) ELAS_DCHECK_DECL(dcheck_eo_p4)
ELAS_DCHECK_DECL(dcheck_eo_p5) ELAS_DCHECK_DECL(dcheck_eo_p6) ELAS_DCHECK_DECL(dcheck_eo_p7) ELAS_DCHECK_DECL(dcheck_eo_p8)
ELAS_DCHECK_DECL(dcheck_simt_p1) ELAS_DCHECK_DECL(dcheck_simt_p2) ELAS_DCHECK_DECL(dcheck_simt_p3) ELAS_DCHECK_DECL(dcheck_simt_p4)
ELAS_DCHECK_DECL(dcheck_simt_p5) ELAS_DCHECK_DECL(dcheck_simt_p6) ELAS_DCHECK_DECL(dcheck_simt_p7) ELAS_DCHECK_DECL(dcheck_simt_p8)
#undef ELAS_DCHECK_DECL

// error helpers
void set_error(const std::string& msg);

// Per-device, thread-safe one-time launch preparation of a kernel: the dynamic shared-memory
// attribute (a per-device function attribute) and the resident-CTA count of the grid
// (SMs x CTAs per SM at this CTA size and shared memory).  One static KernelPrep per kernel
// instance; every launch calls prep() on the current device.
constexpr int kMaxDevices = 64;
struct KernelPrep {
  std::mutex m;
  bool done[kMaxDevices] = {};
  int resident[kMaxDevices] = {};
  template <typename K>
  cudaError_t prep(K kern, int threads, size_t smem, int* resident_ctas) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> g(m);
    if (!done[dev]) {
      if (smem > 48 * 1024) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
      }
      int sms = 0, per_sm = 0;
      if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
      if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem)) != cudaSuccess) return e;
      resident[dev] = sms * (per_sm > 0 ? per_sm : 1);
      done[dev] = true;
    }
    if (resident_ctas) *resident_ctas = resident[dev];
    return cudaSuccess;
  }
};

}  // namespace elas
