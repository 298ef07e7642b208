// One-thread-per-element variant of the fused apply for p = 1 (q = 2 or 3).
//
// At p = 1 an element has 8 nodes and q^3 points; the apply is HBM-bound (qdata dominates:
// 9 q^3 doubles per element against 3 owned dofs), so this variant removes every shared-memory
// transpose and barrier of the fibre kernel: each thread gathers its element, runs the sum
// factorisation line by line in registers (G_xi = D (x) B (x) B, applied one
// x-line of quadrature points at a time -- the "slices" loop order of PAPER.md:315-329 shrunk
// to a line), evaluates the Voigt-symmetric stress at the points, applies the
// transposed contractions and scatters with red.global.add.f64.  Quadrature data is stored
// lane-interleaved over blocks of 32 consecutive elements (QD_LAYOUT_E32), so each of the 9
// loads per point is one fully coalesced 256-byte warp access.
//
// Per x-line (a2, a3):
//   T[c][d][i] = sum_{j,k} Cjk_d[j][k] u[c][k][j][i],   Cjk_0 = By Bz, Cjk_1 = Dy Bz, Cjk_2 = By Dz
//   G[a1][c][d] = sum_i Cx_d[a1][i] T[c][d][i],         Cx_0 = Dx, Cx_1 = Cx_2 = Bx
//   F = pointwise(G, A~, r) at every point of the line
//   S[c][d][i] = sum_a1 Cx_d[a1][i] F[a1][c][d];  out[c][k][j][i] += sum_d Cjk_d[j][k] S[c][d][i]
#include "elas_internal.h"

namespace elas {
namespace lo {

constexpr int NT = 128;
#ifndef ELAS_P1T_MINB
#define ELAS_P1T_MINB 2
#endif

__device__ __forceinline__ bool cons(int I, int J, int K, const Slab& s) {
  const uint32_t f = s.faces;
  return ((f & ELAS_FACE_XMIN) && I == 0) || ((f & ELAS_FACE_XMAX) && I == s.Nx - 1) ||
         ((f & ELAS_FACE_YMIN) && J == 0) || ((f & ELAS_FACE_YMAX) && J == s.Ny - 1) ||
         ((f & ELAS_FACE_ZMIN) && K == 0) || ((f & ELAS_FACE_ZMAX) && K == s.Nz - 1);
}

__device__ __forceinline__ void pointwise(double (&G)[3][3], const double (&A)[9], double r) {
  double H[3][3];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int m = 0; m < 3; ++m) H[c][m] = fma(G[c][2], A[6 + m], fma(G[c][1], A[3 + m], G[c][0] * A[m]));
  const double s = r * (H[0][0] + H[1][1] + H[2][2]);
  double S[3][3];
  S[0][0] = fma(2.0, H[0][0], s);
  S[1][1] = fma(2.0, H[1][1], s);
  S[2][2] = fma(2.0, H[2][2], s);
  S[0][1] = S[1][0] = H[0][1] + H[1][0];
  S[0][2] = S[2][0] = H[0][2] + H[2][0];
  S[1][2] = S[2][1] = H[1][2] + H[2][1];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int d = 0; d < 3; ++d)
      G[c][d] = fma(S[c][2], A[3 * d + 2], fma(S[c][1], A[3 * d + 1], S[c][0] * A[3 * d]));
}

// OTF: geometry on the fly (ELAS_VARIANT_FOLDED_OTF at p = 1): qd = geo32 (QD_LAYOUT_OTF32, 40 words
// per element, lane-interleaved); each thread reads its element's Jacobian/material words per
// x-line (L1-resident after the first) and rebuilds A~ = sqrt(mu) sqrt(w1 w2 w3) adj(J) / sqrt(det)
// at every point: the HBM stream of 9 q^3 doubles per element that bounds this kernel disappears.
template <int Q, bool OTF>
__global__ void __launch_bounds__(NT, ELAS_P1T_MINB)
    apply_p1_kernel(const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ qd,
                    const double* __restrict__ rr, const double* __restrict__ tables, Slab s,
                    int64_t e_begin, int64_t e_end, int pref_ctas, const double* __restrict__ gauss) {
  constexpr int N = 2;
  __shared__ double tb[2 * Q * N + 2 * Q];  // B then D (q x 2): broadcast reads; OTF: g[q], sqrt(w)[q]
  __shared__ double su[24 * NT];     // gathered element vectors, one column per thread
  if (threadIdx.x < 2 * Q * N) tb[threadIdx.x] = tables[threadIdx.x];
  if (OTF && threadIdx.x < 2 * Q) tb[2 * Q * N + threadIdx.x] = gauss[threadIdx.x];
#if ELAS_L2_PREFETCH
  if (!OTF && threadIdx.x == 0 && pref_ctas > 0) {
    const int64_t pe0 = e_begin + ((int64_t)blockIdx.x + pref_ctas) * NT;
    if (pe0 < e_end) {
      const int64_t pne = (e_end - pe0) < NT ? (e_end - pe0) : NT;
      const int64_t blocks = (pne + 31) / 32;
      const uintptr_t a0 = (uintptr_t)(qd + (pe0 / 32) * (int64_t)(32 * 9 * Q * Q * Q));
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0),
                   "r"((uint32_t)(blocks * 32 * 9 * Q * Q * Q * 8)) : "memory");
    }
  }
#endif
  __syncthreads();
  const int64_t e = e_begin + (int64_t)blockIdx.x * NT + threadIdx.x;
  if (e >= e_end) return;
  const double* TB = tb;
  const double* TD = tb + Q * N;
  const int ex = (int)(e % s.nx), ey = (int)((e / s.nx) % s.ny), ez = (int)(e / ((int64_t)s.nx * s.ny));
  const int64_t plane = (int64_t)s.Nx * s.Ny;
  const int64_t base = ex + (int64_t)s.Nx * ey + plane * ez;  // p = 1: node (ex, ey, ez)
  const bool bc = s.faces != 0;

  // gather (Dirichlet dofs zeroed) into this thread's column of shared memory:
  // su[v][tid], v = c*8 + k*4 + j*2 + i (conflict-free: consecutive threads, consecutive words)
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const bool z = bc && cons(ex + i, ey + j, ez + k, s);
        const int64_t o = base + i + (int64_t)s.Nx * j + plane * k;
        ELAS_DCHECK(o >= 0 && 2 * s.nodes + o < 3 * s.nodes);
#pragma unroll
        for (int c = 0; c < 3; ++c) su[(c * 8 + k * 4 + j * 2 + i) * NT + threadIdx.x] = z ? 0.0 : __ldg(x + c * s.nodes + o);
      }
  double out[3][2][2][2];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int i = 0; i < 2; ++i) out[c][k][j][i] = 0.0;

  const double r = __ldg(rr + e);
  const int lane = (int)(e & 31);
  const double* qb = qd + (e >> 5) * (int64_t)(32 * 9 * Q * Q * Q) + lane;
  // OTF: this element's geometry words, read per line through L1 (coalesced, lane-interleaved)
  const double* gcol = qd + (e >> 5) * (int64_t)(32 * GEO_WORDS) + lane;
  constexpr int GS = 32;
  const double* gq = tb + 2 * Q * N;   // Gauss points, then sqrt weights (OTF)

#pragma unroll 1
  for (int a3 = 0; a3 < Q; ++a3)
#pragma unroll 1
    for (int a2 = 0; a2 < Q; ++a2) {
      double cjk[3][2][2];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          cjk[0][j][k] = TB[a2 * N + j] * TB[a3 * N + k];
          cjk[1][j][k] = TD[a2 * N + j] * TB[a3 * N + k];
          cjk[2][j][k] = TB[a2 * N + j] * TD[a3 * N + k];
        }
      double G[Q][3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          double T[2];
          const double* uc = su + c * 8 * NT + threadIdx.x;   // u[c][k][j][i] at uc[(4k + 2j + i) NT]
#pragma unroll
          for (int i = 0; i < 2; ++i)
            T[i] = fma(cjk[d][1][1], uc[(6 + i) * NT],     // (j, k) = (1, 1)
                       fma(cjk[d][1][0], uc[(2 + i) * NT],   // (j, k) = (1, 0)
                           fma(cjk[d][0][1], uc[(4 + i) * NT], cjk[d][0][0] * uc[i * NT])));
          const double* cx = d == 0 ? TD : TB;
#pragma unroll
          for (int a1 = 0; a1 < Q; ++a1) G[a1][c][d] = fma(cx[a1 * N + 1], T[1], cx[a1 * N] * T[0]);
        }
      if constexpr (OTF) {
        // per line: dx/dxi1 constant, dx/dxi2 and dx/dxi3 linear in xi1
        const double xi2 = gq[a2], xi3 = gq[a3];
        double col1[3], b2[3], s2[3], b3[3], s3[3];
#pragma unroll
        for (int m = 0; m < 3; ++m) {
          col1[m] = fma(fma(__ldg(gcol + (9 + m) * GS), xi3, __ldg(gcol + (3 + m) * GS)), xi2, fma(__ldg(gcol + (6 + m) * GS), xi3, __ldg(gcol + m * GS)));
          b2[m] = fma(__ldg(gcol + (18 + m) * GS), xi3, __ldg(gcol + (12 + m) * GS));
          s2[m] = fma(__ldg(gcol + (21 + m) * GS), xi3, __ldg(gcol + (15 + m) * GS));
          b3[m] = fma(__ldg(gcol + (30 + m) * GS), xi2, __ldg(gcol + (24 + m) * GS));
          s3[m] = fma(__ldg(gcol + (33 + m) * GS), xi2, __ldg(gcol + (27 + m) * GS));
        }
        const double sq = __ldg(gcol + 36 * GS) * gq[Q + a2] * gq[Q + a3];
#pragma unroll
        for (int a1 = 0; a1 < Q; ++a1) {
          const double xi1 = gq[a1];
          double J[3][3];
#pragma unroll
          for (int m = 0; m < 3; ++m) {
            J[m][0] = col1[m];
            J[m][1] = fma(s2[m], xi1, b2[m]);
            J[m][2] = fma(s3[m], xi1, b3[m]);
          }
          double adj[3][3];
          adj[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
          adj[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
          adj[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
          adj[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
          adj[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
          adj[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
          adj[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
          adj[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
          adj[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
          const double det = J[0][0] * adj[0][0] + J[0][1] * adj[1][0] + J[0][2] * adj[2][0];
          const double sc = sq * gq[Q + a1] * rsqrt(det);
          double A[9];
#pragma unroll
          for (int d = 0; d < 3; ++d)
#pragma unroll
            for (int m = 0; m < 3; ++m) A[3 * d + m] = sc * adj[d][m];
          pointwise(G[a1], A, r);
        }
      } else {
#pragma unroll
        for (int a1 = 0; a1 < Q; ++a1) {
          const double* q = qb + (int64_t)((a1 + Q * (a2 + Q * a3)) * 9) * 32;
          double A[9];
#pragma unroll
          for (int f = 0; f < 9; ++f) A[f] = __ldg(q + f * 32);
          pointwise(G[a1], A, r);
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double* cx = d == 0 ? TD : TB;
          double S[2] = {0.0, 0.0};
#pragma unroll
          for (int a1 = 0; a1 < Q; ++a1) {
            S[0] = fma(cx[a1 * N], G[a1][c][d], S[0]);
            S[1] = fma(cx[a1 * N + 1], G[a1][c][d], S[1]);
          }
#pragma unroll
          for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int i = 0; i < 2; ++i) out[c][k][j][i] = fma(cjk[d][j][k], S[i], out[c][k][j][i]);
        }
    }

#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        if (bc && cons(ex + i, ey + j, ez + k, s)) continue;
        const int64_t o = base + i + (int64_t)s.Nx * j + plane * k;
        ELAS_DCHECK(o >= 0 && 2 * s.nodes + o < 3 * s.nodes);
#pragma unroll
        for (int c = 0; c < 3; ++c) atomicAdd(y + c * s.nodes + o, out[c][k][j][i]);
      }
}

template <int Q, bool OTF>
cudaError_t launch_q(const Slab& s, const double* x, double* y, const double* qd, const double* rr,
                     const double* tables, int64_t e_begin, int64_t e_end, cudaStream_t st, const double* gauss) {
  static KernelPrep prep;   // per device
  int pref = 0;
  cudaError_t e = prep.prep(apply_p1_kernel<Q, OTF>, NT, 0, &pref);
  if (e != cudaSuccess) return e;
  const int64_t ne = e_end - e_begin;
  if (ne <= 0) return cudaSuccess;
  const int64_t grid = (ne + NT - 1) / NT;
  apply_p1_kernel<Q, OTF><<<(unsigned)grid, NT, 0, st>>>(x, y, qd, rr, tables, s, e_begin, e_end, pref, gauss);
  return cudaGetLastError();
}

}  // namespace lo

cudaError_t apply_p1t_launch(int q, const Slab& s, const double* x, double* y, const double* qd, const double* rr,
                             const double* tables, int64_t e_begin, int64_t e_end, cudaStream_t st, int otf) {
  const double* gauss = tables + tables_gauss_offset(1, q, fold_table_size(1, q));
  if (q == 2) return otf ? lo::launch_q<2, true>(s, x, y, qd, rr, tables, e_begin, e_end, st, gauss)
                         : lo::launch_q<2, false>(s, x, y, qd, rr, tables, e_begin, e_end, st, gauss);
  if (q == 3) return otf ? lo::launch_q<3, true>(s, x, y, qd, rr, tables, e_begin, e_end, st, gauss)
                         : lo::launch_q<3, false>(s, x, y, qd, rr, tables, e_begin, e_end, st, gauss);
  return cudaErrorInvalidValue;
}

}  // namespace elas

ELAS_DCHECK_READER(dcheck_p1t)
