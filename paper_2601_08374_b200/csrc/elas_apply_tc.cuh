// FP64 tensor-core (mma.sync.m16n8k4.f64, SASS DMMA) variant of the fused apply kernel for
// p = 6, q = 8 (n = 7 nodes, 8 points per direction) -- the degree of configs 3 and 5 and the
// paper's throughput sweet spot.
//
// Same operator and stage semantics as elas_apply.cuh (gather, forward sum factorisation,
// Voigt-symmetric pointwise stress, transposed sum factorisation, scatter-add); only the 1D
// contractions run on the FP64 tensor path.  Every 1D contraction over a length-7 (nodes) or
// length-8 (points) index is a [16 fibres x K] x [K x 8] MMA: fibres are the M rows, the
// contracted index is K (7 padded to 8 with zero coefficients), the produced index the 8
// columns.  Coefficient fragments (B, D and their transposes) live in registers for the whole
// kernel.  A PAIR OF WARPS processes one element; the warp's shared-memory tiles are bounded by
// processing the y/z stages in four slices of two x-points (a1), the GPU form of the paper's
// "fibers to slices" loop structure.  Two warps share an element: each
// does half of the x-stage tiles, two of the four slices, and half of the x-transpose tiles.
//
// Fragment layouts (verified on B200 by tools/microbench/dmma_layout.cu), g = lane>>2, t = lane&3:
//   A 16x4: a0 = A[g][t], a1 = A[g+8][t];  B 4x8: b0 = B[t][g];
//   C 16x8: c0 = C[g][2t], c1 = C[g][2t+1], c2 = C[g+8][2t], c3 = C[g+8][2t+1].
//
// Per element (e):
//   XF  fibres (c,j,k), K=i      : UX[c][0] = Bx u, UX[c][1] = Dx u          (global x -> smem UX)
//   for each a1-slice s (a1 = 2s, 2s+1):
//     YF  fibres (k,a1), K=j     : w0=(Dx,By)=By UX1, w1=(Bx,Dy)=Dy UX0, w2=(Bx,By)=By UX0 (UX -> U2)
//     ZF  fibres (a1,a2), K=k    : G[c][d] = (Bz w0, Bz w1, Dz w2) at (a1,a2,a3)   (U2 -> registers)
//     pointwise on the C fragments (qdata streamed from HBM in fragment order)
//     ZB  K=a3 (C->A register reuse with a permuted K order)                 (registers -> U2)
//     YB  fibres (k,a1), K=a2    : T0 = By^T V0, T1 = Dy^T V1 + By^T V2      (U2 -> UX, in place)
//   XB  fibres (c,j,k), K=a1     : y += Dx^T T0 + Bx^T T1                    (UX -> red.global)
#pragma once
#include "elas_internal.h"

namespace elas {
namespace tc {

constexpr int P = 6, Q = 8, N = 7;
constexpr int NSLICE = 4;
// UX[c][v][k][j][a1]: 7 x 8 (j, a1) rows per k, unpadded; a1 XOR-swizzled by (j, k) so that the
// x-stage pair stores, the y-stage fragment loads and the x-transpose fragment loads are all
// bank-conflict free (16 distinct double-word banks per half-warp).
constexpr int UX_J = 8, UX_K = N * UX_J, UX_V = N * UX_K, UX_C = 2 * UX_V, UX_SIZE = 3 * UX_C;
// U2[c][w][k][a1l][a2] per slice: a2 XOR-swizzled by k, a1l XOR-swizzled by k so the fragment
// loads of the z stage cover 16 distinct banks.
constexpr int U2_A = 8, U2_K = 2 * U2_A, U2_W = N * U2_K, U2_C = 3 * U2_W, U2_SIZE = 3 * U2_C;
#ifndef ELAS_TC_EPC
#define ELAS_TC_EPC 6
#endif
constexpr int EPC = ELAS_TC_EPC;               // elements per CTA, two warps each
constexpr int ELEM_SMEM = UX_SIZE + 2 * U2_SIZE;  // doubles per element (one U2 per warp)
constexpr int QD_PER_ELEM = 9 * Q * Q * Q;     // 4608 doubles, fragment order (see qdata kernel)

__device__ __forceinline__ int ux(int c, int v, int k, int j, int a1) {
  return c * UX_C + v * UX_V + k * UX_K + j * UX_J + (a1 ^ ((((j >> 1) & 1) << 2) | ((k & 1) << 1)));
}
__device__ __forceinline__ int u2(int c, int w, int k, int a1l, int a2) {
  return c * U2_C + w * U2_W + k * U2_K + ((a1l ^ ((k >> 1) & 1)) << 3) + (a2 ^ (((k ^ (k >> 2)) & 1) << 2));
}

__device__ __forceinline__ void mma(double (&c)[4], double a0, double a1, double b) {
  asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

__device__ __forceinline__ bool cons(int I, int J, int K, const Slab& s) {
  const uint32_t f = s.faces;
  return ((f & ELAS_FACE_XMIN) && I == 0) || ((f & ELAS_FACE_XMAX) && I == s.Nx - 1) ||
         ((f & ELAS_FACE_YMIN) && J == 0) || ((f & ELAS_FACE_YMAX) && J == s.Ny - 1) ||
         ((f & ELAS_FACE_ZMIN) && K == 0) || ((f & ELAS_FACE_ZMAX) && K == s.Nz - 1);
}

// sigma~ = r tr(H) I + H + H^T, H = G A~; F = sigma~ A~^T  (Voigt-symmetric, 6 unique)
__device__ __forceinline__ void pointwise(double (&G)[3][3], const double* A, double r) {
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

// Named barrier for the two warps of element `el` (ids 1..EPC; 0 is __syncthreads).
__device__ __forceinline__ void pair_sync(int el) {
  asm volatile("bar.sync %0, 64;" ::"r"(el + 1) : "memory");
}

// fibre f of the x stages -> (c, j, k), f = c*49 + k*7 + j
__device__ __forceinline__ void fibre(int f, int& c, int& j, int& k) {
  const int fc = f < 3 * N * N ? f : 0;
  c = fc / (N * N);
  const int r = fc % (N * N);
  j = r % N;
  k = r / N;
}

__global__ void __launch_bounds__(64 * EPC, 1)
    apply_tc_kernel(const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ qd,
                    const double* __restrict__ rr, const double* __restrict__ tables, Slab s,
                    int64_t e_begin, int64_t e_end, int pref_ctas) {
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int el = warp >> 1, half = warp & 1;
  const int g = lane >> 2, t = lane & 3;
  const int64_t cta_e0 = e_begin + (int64_t)blockIdx.x * EPC;
  const int64_t e = cta_e0 + el;
#if ELAS_L2_PREFETCH
  if (threadIdx.x == 0 && pref_ctas > 0) {
    // TMA bulk prefetch into L2 of the qdata of the CTA one wave ahead
    const int64_t pe0 = cta_e0 + (int64_t)pref_ctas * EPC;
    if (pe0 < e_end) {
      const int64_t pne = (e_end - pe0) < EPC ? (e_end - pe0) : EPC;
      const uintptr_t a0 = (uintptr_t)(qd + pe0 * (int64_t)QD_PER_ELEM);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0),
                   "r"((uint32_t)(pne * QD_PER_ELEM * 8)) : "memory");
    }
  }
#endif
  if (e >= e_end) return;  // both warps of an element exit together
  double* UX = smem + el * ELEM_SMEM;
  double* U2 = UX + UX_SIZE + half * U2_SIZE;

  // coefficient fragments (registers, whole kernel).  tables = B[a][i] (Q x N) then D.
  const double* TB = tables;
  const double* TD = tables + Q * N;
  double FB[2], FD[2], BB[2], BD[2], BBp[2], BDp[2];
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    const int i = 4 * ks + t;                 // forward: K = node index, column = point g
    FB[ks] = i < N ? __ldg(TB + g * N + i) : 0.0;
    FD[ks] = i < N ? __ldg(TD + g * N + i) : 0.0;
    const int a = 4 * ks + t;                 // backward: K = point index, column = node g
    BB[ks] = g < N ? __ldg(TB + a * N + g) : 0.0;
    BD[ks] = g < N ? __ldg(TD + a * N + g) : 0.0;
    const int ap = 2 * t + ks;                // permuted K order of the fused z stage
    BBp[ks] = g < N ? __ldg(TB + ap * N + g) : 0.0;
    BDp[ks] = g < N ? __ldg(TD + ap * N + g) : 0.0;
  }

  const int ex = (int)(e % s.nx), ey = (int)((e / s.nx) % s.ny), ez = (int)(e / ((int64_t)s.nx * s.ny));
  const int64_t plane = (int64_t)s.Nx * s.Ny;
  const bool bc = s.faces != 0;
  const int I0 = ex * P, J0 = ey * P, K0 = ez * P;
  const int64_t ebase = I0 + (int64_t)s.Nx * J0 + plane * K0;

  // ---------------- XF: gather + contraction in x (tiles T = half, half+2, ...) ----------
  {
    double a[5][2][2];  // all gathers of this warp issued before any MMA
#pragma unroll
    for (int u = 0; u < 5; ++u)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int f = 16 * (2 * u + half) + g + 8 * h;
        int c, j, k;
        fibre(f, c, j, k);
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const int i = 4 * ks + t;
          double v = 0.0;
          if (f < 3 * N * N && i < N && !(bc && cons(I0 + i, J0 + j, K0 + k, s)))
            v = __ldg(x + c * s.nodes + ebase + i + (int64_t)s.Nx * j + plane * k);
          a[u][ks][h] = v;
        }
      }
#pragma unroll
    for (int u = 0; u < 5; ++u) {
      double cb[4] = {0, 0, 0, 0}, cd[4] = {0, 0, 0, 0};
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        mma(cb, a[u][ks][0], a[u][ks][1], FB[ks]);
        mma(cd, a[u][ks][0], a[u][ks][1], FD[ks]);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int f = 16 * (2 * u + half) + g + 8 * h;
        if (f < 3 * N * N) {
          int c, j, k;
          fibre(f, c, j, k);
          *reinterpret_cast<double2*>(UX + ux(c, 0, k, j, 2 * t)) = make_double2(cb[2 * h], cb[2 * h + 1]);
          *reinterpret_cast<double2*>(UX + ux(c, 1, k, j, 2 * t)) = make_double2(cd[2 * h], cd[2 * h + 1]);
        }
      }
    }
  }
  pair_sync(el);

  const double re = __ldg(rr + e);
  const double* qe = qd + e * (int64_t)QD_PER_ELEM;

#pragma unroll 1
  for (int ss = 0; ss < 2; ++ss) {
    const int sl = 2 * half + ss;   // this warp's slices: a1 in {2 sl, 2 sl + 1}
    // qdata of this slice: 4 points x 9 values per lane, issued early (consumed after ZF)
    double Aq[4][9];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int f = 0; f < 9; ++f) Aq[r][f] = __ldg(qe + ((sl * 4 + r) * 9 + f) * 32 + lane);

    // ---------------- YF: contraction in y (fibres ff = 2k + a1l, 14 of 16 rows) ---------
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double a0[2][2], a1v[2][2];  // [ks][row h] of UX0 (Bx) and UX1 (Dx)
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int ff = g + 8 * h, k = ff >> 1, a1l = ff & 1;
          const int j = 4 * ks + t;
          const bool ok = ff < 2 * N && j < N;
          a0[ks][h] = ok ? UX[ux(c, 0, k, j, 2 * sl + a1l)] : 0.0;
          a1v[ks][h] = ok ? UX[ux(c, 1, k, j, 2 * sl + a1l)] : 0.0;
        }
      double w0[4] = {0, 0, 0, 0}, w1[4] = {0, 0, 0, 0}, w2[4] = {0, 0, 0, 0};
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        mma(w0, a1v[ks][0], a1v[ks][1], FB[ks]);  // (Dx, By)
        mma(w1, a0[ks][0], a0[ks][1], FD[ks]);    // (Bx, Dy)
        mma(w2, a0[ks][0], a0[ks][1], FB[ks]);    // (Bx, By)
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int ff = g + 8 * h, k = ff >> 1, a1l = ff & 1;
        if (ff < 2 * N) {
          *reinterpret_cast<double2*>(U2 + u2(c, 0, k, a1l, 2 * t)) = make_double2(w0[2 * h], w0[2 * h + 1]);
          *reinterpret_cast<double2*>(U2 + u2(c, 1, k, a1l, 2 * t)) = make_double2(w1[2 * h], w1[2 * h + 1]);
          *reinterpret_cast<double2*>(U2 + u2(c, 2, k, a1l, 2 * t)) = make_double2(w2[2 * h], w2[2 * h + 1]);
        }
      }
    }
    __syncwarp();

    // ---------------- ZF: contraction in z -> gradients in C fragments -----------------
    // rows: phi = g -> (a1l 0, a2 g), phi = g+8 -> (a1l 1, a2 g); cols a3 = 2t, 2t+1
    double G[3][3][4];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int w = 0; w < 3; ++w) {
        double acc[4] = {0, 0, 0, 0};
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const int k = 4 * ks + t;
          const double v0 = k < N ? U2[u2(c, w, k, 0, g)] : 0.0;
          const double v1 = k < N ? U2[u2(c, w, k, 1, g)] : 0.0;
          mma(acc, v0, v1, w == 2 ? FD[ks] : FB[ks]);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) G[c][w][r] = acc[r];
      }

    // ---------------- pointwise on the fragments -------------------------------------
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      double Gp[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) Gp[c][d] = G[c][d][r];
      pointwise(Gp, Aq[r], re);
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) G[c][d][r] = Gp[c][d];
    }
    __syncwarp();  // all lanes finished reading U2 before it is overwritten

    // ---------------- ZB: transposed z, A operand straight from the C fragments ---------
    // K position (ks, t) <-> a3 = 2t + ks: ks = 0 uses c0/c2, ks = 1 uses c1/c3
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        double v[4] = {0, 0, 0, 0};
        mma(v, G[c][d][0], G[c][d][2], d == 2 ? BDp[0] : BBp[0]);
        mma(v, G[c][d][1], G[c][d][3], d == 2 ? BDp[1] : BBp[1]);
        // rows phi (a1l = h, a2 = g), cols k = 2t, 2t+1
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          U2[u2(c, d, 2 * t, h, g)] = v[2 * h];
          if (2 * t + 1 < N) U2[u2(c, d, 2 * t + 1, h, g)] = v[2 * h + 1];
        }
      }
    __syncwarp();

    // ---------------- YB: transposed y -> T0, T1 into UX (this slice's a1 columns) ------
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double t0[4] = {0, 0, 0, 0}, t1[4] = {0, 0, 0, 0};
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        double v0[2], v1[2], v2[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int ff = g + 8 * h, k = ff >> 1, a1l = ff & 1;
          const int a2 = 4 * ks + t;
          const bool ok = ff < 2 * N;
          v0[h] = ok ? U2[u2(c, 0, k, a1l, a2)] : 0.0;
          v1[h] = ok ? U2[u2(c, 1, k, a1l, a2)] : 0.0;
          v2[h] = ok ? U2[u2(c, 2, k, a1l, a2)] : 0.0;
        }
        mma(t0, v0[0], v0[1], BB[ks]);   // By^T V0
        mma(t1, v1[0], v1[1], BD[ks]);   // Dy^T V1
        mma(t1, v2[0], v2[1], BB[ks]);   // + By^T V2
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int ff = g + 8 * h, k = ff >> 1, a1l = ff & 1;
        if (ff < 2 * N) {
          UX[ux(c, 0, k, 2 * t, 2 * sl + a1l)] = t0[2 * h];
          UX[ux(c, 1, k, 2 * t, 2 * sl + a1l)] = t1[2 * h];
          if (2 * t + 1 < N) {
            UX[ux(c, 0, k, 2 * t + 1, 2 * sl + a1l)] = t0[2 * h + 1];
            UX[ux(c, 1, k, 2 * t + 1, 2 * sl + a1l)] = t1[2 * h + 1];
          }
        }
      }
    }
    __syncwarp();
  }
  pair_sync(el);

  // ---------------- XB: transposed x + scatter-add (tiles T = half, half+2, ...) ---------
#pragma unroll
  for (int u = 0; u < 5; ++u) {
    const int T = 2 * u + half;
    int cc[2], jj[2], kk[2];
    bool okr[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int f = 16 * T + g + 8 * h;
      okr[h] = f < 3 * N * N;
      fibre(f, cc[h], jj[h], kk[h]);
    }
    double o[4] = {0, 0, 0, 0};
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int a1 = 4 * ks + t;
      double p0[2], p1[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        p0[h] = okr[h] ? UX[ux(cc[h], 0, kk[h], jj[h], a1)] : 0.0;
        p1[h] = okr[h] ? UX[ux(cc[h], 1, kk[h], jj[h], a1)] : 0.0;
      }
      mma(o, p0[0], p0[1], BD[ks]);   // Dx^T T0
      mma(o, p1[0], p1[1], BB[ks]);   // Bx^T T1
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!okr[h]) continue;
#pragma unroll
      for (int uu = 0; uu < 2; ++uu) {
        const int i = 2 * t + uu;
        if (i >= N) continue;
        if (bc && cons(I0 + i, J0 + jj[h], K0 + kk[h], s)) continue;
        atomicAdd(y + cc[h] * s.nodes + ebase + i + (int64_t)s.Nx * jj[h] + plane * kk[h], o[2 * h + uu]);
      }
    }
  }
}

}  // namespace tc
}  // namespace elas
