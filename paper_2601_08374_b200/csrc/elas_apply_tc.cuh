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
// Even-odd folding where one input feeds two tables (GLL/Gauss symmetry, elas_apply_eo.cuh):
// XF contracts u+ = u_i + u_{6-i} and u- = u_i - u_{6-i} (K = 4 node pairs) against the folded
// [B | D] tables in one E and one O MMA (2 instead of 4 per tile), and YF does the same for the
// two y-contractions of UX0 (w1 = Dy UX0, w2 = By UX0: 2 instead of 4 MMAs per component);
// out_a = E + O, out_{7-a} = +-(E - O).  The single-table contractions (ZF, ZB, YB, XB, w0)
// gain nothing from folding on the tensor path and stay plain.
//
// Persistent element slots: the grid covers the SMs, each slot (WPE warps) walks the elements
// e0 + el, e0 + el + EPC gridDim, ... with its own named barrier, and at the start of each
// element pulls the NEXT element's x rows and quadrature data into L2 (prefetch.global.L2 and
// one cp.async.bulk.prefetch.L2), so the global loads of the next XF and slices hit L2.
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
#define ELAS_TC_EPC 4   // measured (config 4, p6): 4 -> 31.4, 5 -> 25.0, 6 -> 28.3 GDoF/s (6, 5: 168 regs + spills)
#endif
#ifndef ELAS_TC_WPE
#define ELAS_TC_WPE 2
#endif
constexpr int EPC = ELAS_TC_EPC;               // elements per CTA
constexpr int WPE = ELAS_TC_WPE;               // warps per element (2 or 4): slices split between them
constexpr int ELEM_SMEM = UX_SIZE + WPE * U2_SIZE;  // doubles per element (one U2 per warp)
constexpr int XTILES = (3 * N * N + 15) / 16;       // 10 fibre tiles in the x stages
constexpr int XT_PER_WARP = (XTILES + WPE - 1) / WPE;
static_assert(NSLICE % WPE == 0, "slices must split evenly over the warps of an element");
constexpr int QD_PER_ELEM = 9 * Q * Q * Q;     // 4608 doubles, fragment order (see qdata kernel)
constexpr int FTS = 4 * N + 4 * Q;             // doubles per folded table (fold_table_size(6, 8))

// swizzled offsets inside one (c, v) block of UX / one (c, w) block of U2
__device__ __forceinline__ int uxo(int k, int j, int a1) {
  return k * UX_K + j * UX_J + (a1 ^ ((((j >> 1) & 1) << 2) | ((k & 1) << 1)));
}
__device__ __forceinline__ int u2o(int k, int a1l, int a2) {
  return k * U2_K + ((a1l ^ ((k >> 1) & 1)) << 3) + (a2 ^ (((k ^ (k >> 2)) & 1) << 2));
}

__device__ __forceinline__ void mma(double (&c)[4], double a0, double a1, double b) {
  asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

// 8-row variant (SASS: one DMMA.8x8x4): a0 = A[g][t], b0 = B[t][g], c0/c1 = C[g][2t], C[g][2t+1]
__device__ __forceinline__ void mma8(double (&c)[2], double a0, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a0), "d"(b));
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

// Named barrier for the WPE warps of element `el` (ids 1..EPC; 0 is __syncthreads).
__device__ __forceinline__ void pair_sync(int el) {
  asm volatile("bar.sync %0, %1;" ::"r"(el + 1), "r"(32 * WPE) : "memory");
}

// fibre f of the x stages -> (c, j, k), f = c*49 + k*7 + j; rows past the last fibre are
// clamped onto it (their results are never stored; padding columns meet zero coefficients)
__device__ __forceinline__ void fibre(int f, int& c, int& j, int& k) {
  const int fc = f < 3 * N * N ? f : 3 * N * N - 1;
  c = fc / (N * N);
  const int r = fc - c * (N * N);
  k = r / N;
  j = r - k * N;
}

__global__ void __launch_bounds__(32 * WPE * EPC, 1)
    apply_tc_kernel(const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ qd,
                    const double* __restrict__ rr, const double* __restrict__ tables, Slab s,
                    int64_t e_begin, int64_t e_end) {
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int el = warp / WPE, half = warp % WPE;   // `half`: this warp's index within its element
  const int g = lane >> 2, t = lane & 3;
  double* UX = smem + el * ELEM_SMEM;
  double* U2 = UX + UX_SIZE + half * U2_SIZE;

  // coefficient fragments (registers, whole kernel).  tables = B[a][i] (Q x N), D, fold(B), fold(D)
  const double* TB = tables;
  const double* TD = tables + Q * N;
  double FB[2], BB[2], BD[2], BBp[2], BDp[2], FD[2];
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
  // folded fragments (E and O MMAs of XF / YF): row k = t = node pair (t < 3: (t, 6 - t); t = 3:
  // the middle node), column n = g: n < 4 the B pair a = n, n >= 4 the D pair a = n - 4
  const double* fB = tables + 2 * Q * N;
  const double* fD = fB + FTS;
  const double FEf = g < 4 ? __ldg(fB + g * 4 + t) : __ldg(fD + (g - 4) * 4 + t);
  const double FOf = t < 3 ? (g < 4 ? __ldg(fB + 16 + g * 3 + t) : __ldg(fD + 16 + (g - 4) * 3 + t)) : 0.0;

  const int64_t plane = (int64_t)s.Nx * s.Ny;
  const bool bc = s.faces != 0;
  // lane constants of the slice stages (rows ff = g + 8h -> k = ff >> 1, a1l = ff & 1)
  const int gl = g & 1, gh = g >> 1;
  const int kr[2] = {gh, (gh + 4) < N ? gh + 4 : N - 1};
  const bool row1 = g + 8 < 2 * N;
  const int sw_yb = ((t & 1) << 2) | ((gh & 1) << 1);         // UX swizzle of (j = 2t+u, k = kr[h])
  const int iK[2] = {t, (4 + t) < N ? 4 + t : N - 1};   // K index 4 ks + t, clamped (zero coefficient)
  int yfb[2][2], ybl[2][2], zfl[2][2], zbs[2][2], ybs[2][2], yfs[2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      yfb[a][h] = kr[h] * UX_K + iK[a] * UX_J + gl;          // YF load (w0), a = ks
      ybl[a][h] = u2o(kr[h], gl, 4 * a + t);                   // YB load, a = ks
      zfl[a][h] = u2o(iK[a], h, g);                            // ZF load, a = ks
      zbs[a][h] = u2o((2 * t + a) < N ? 2 * t + a : N - 1, h, g);  // ZB store, a = u (k = 2t+u)
      ybs[a][h] = kr[h] * UX_K + (2 * t + a) * UX_J + gl;      // YB store, a = u (j = 2t+u)
    }
#pragma unroll
  for (int h = 0; h < 2; ++h) yfs[h] = u2o(kr[h], gl, 2 * t);
  const int jlo = t, jhi = 6 - t;                              // folded node pair of this lane

  const int64_t stride = (int64_t)gridDim.x * EPC;
  for (int64_t e = e_begin + (int64_t)blockIdx.x * EPC + el; e < e_end; e += stride) {
    pair_sync(el);   // the previous element's XB is done with UX
    const int ex = (int)(e % s.nx), ey = (int)((e / s.nx) % s.ny), ez = (int)(e / ((int64_t)s.nx * s.ny));
    const int I0 = ex * P, J0 = ey * P, K0 = ez * P;
    const int64_t ebase = I0 + (int64_t)s.Nx * J0 + plane * K0;
    const double* qe = qd + e * (int64_t)QD_PER_ELEM;
#if ELAS_L2_PREFETCH
    {  // the slot's NEXT element: quadrature data (one bulk prefetch) and x rows into L2
      const int64_t en = e + stride;
      if (en < e_end) {
        if (lane == 0 && half == 0)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(qd + en * (int64_t)QD_PER_ELEM),
                       "r"((uint32_t)(QD_PER_ELEM * 8)) : "memory");
        const int nx_ = (int)(en % s.nx), ny_ = (int)((en / s.nx) % s.ny), nz_ = (int)(en / ((int64_t)s.nx * s.ny));
        const int64_t nbase = nx_ * P + (int64_t)s.Nx * (ny_ * P) + plane * (nz_ * P);
#pragma unroll
        for (int u = 0; u < XT_PER_WARP; ++u)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (t == 0) {   // one lane per fibre row (a row is 56 B)
              int c, j, k;
              fibre(16 * (WPE * u + half) + g + 8 * h, c, j, k);
              const double* src = x + c * s.nodes + nbase + (int64_t)s.Nx * j + plane * k;
              asm volatile("prefetch.global.L2 [%0];" ::"l"(src));
              asm volatile("prefetch.global.L2 [%0];" ::"l"(src + N - 1));
            }
          }
      }
    }
#endif

    // ---------------- XF: gather + folded contraction in x (tiles T = half, half+2, ...) -----
    {
      double up[XT_PER_WARP][2], um[XT_PER_WARP][2];  // [tile][h]: all gathers issued before any MMA
#pragma unroll
      for (int u = 0; u < XT_PER_WARP; ++u)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int c, j, k;
          fibre(16 * (WPE * u + half) + g + 8 * h, c, j, k);
          const double* src = x + c * s.nodes + ebase + (int64_t)s.Nx * j + plane * k;
          ELAS_DCHECK(src >= x && (src - x) + N - 1 < 3 * s.nodes);
          double lo = __ldg(src + jlo), hi = __ldg(src + jhi);
          if (bc) {
            if (cons(I0 + jlo, J0 + j, K0 + k, s)) lo = 0.0;
            if (cons(I0 + jhi, J0 + j, K0 + k, s)) hi = 0.0;
          }
          up[u][h] = t < 3 ? lo + hi : lo;
          um[u][h] = t < 3 ? lo - hi : 0.0;
        }
#pragma unroll
      for (int u = 0; u < XT_PER_WARP; ++u) {
        if (WPE * u + half >= XTILES) break;
        double cE[4] = {0, 0, 0, 0}, cO[4] = {0, 0, 0, 0};
        mma(cE, up[u][0], up[u][1], FEf);
        mma(cO, um[u][0], um[u][1], FOf);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int f = 16 * (WPE * u + half) + g + 8 * h;
          if (f < 3 * N * N) {
            int c, j, k;
            fibre(f, c, j, k);
            const int tab = t >> 1;                    // column pair 2t, 2t+1 -> table, pairs a
            double* dst = UX + c * UX_C + tab * UX_V;
#pragma unroll
            for (int uu = 0; uu < 2; ++uu) {
              const int a = 2 * (t & 1) + uu;
              const double E = cE[2 * h + uu], O = cO[2 * h + uu];
              dst[uxo(k, j, a)] = E + O;
              dst[uxo(k, j, 7 - a)] = tab == 0 ? E - O : O - E;
            }
          }
        }
      }
    }
    pair_sync(el);

    const double re = __ldg(rr + e);

#pragma unroll 1
    for (int ss = 0; ss < NSLICE / WPE; ++ss) {
      const int sl = (NSLICE / WPE) * half + ss;   // this warp's slices: a1 in {2 sl, 2 sl + 1}
      const int sw_yf = (((t >> 1) & 1) << 2) | ((gh & 1) << 1);
      const int xyf = (2 * sl) ^ sw_yf, xyb = (2 * sl) ^ sw_yb;
      const double* qs = qe + sl * 4 * 9 * 32 + lane;   // qdata of this slice, fragment order
      // rows h = 0 of the fused z stage: qdata of points r = 0, 1 requested before the y stage
      double Aq[2][9];
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int f = 0; f < 9; ++f) Aq[r][f] = __ldg(qs + (r * 9 + f) * 32);

      // ---------------- YF: contraction in y (fibres ff = 2k + a1l, 14 of 16 rows) ---------
      {
        double dx[3][2][2];             // [c][ks][h]: UX1 = Dx u (plain, K = j)
        double bp[3][2], bm[3][2];      // [c][h]: UX0 = Bx u folded over j (K = node pair)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
#pragma unroll
            for (int h = 0; h < 2; ++h) dx[c][ks][h] = UX[c * UX_C + UX_V + xyf + yfb[ks][h]];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int a1 = 2 * sl + gl;
            const double lo = UX[c * UX_C + uxo(kr[h], jlo, a1)];
            const double hi = UX[c * UX_C + uxo(kr[h], jhi, a1)];
            bp[c][h] = t < 3 ? lo + hi : lo;
            bm[c][h] = t < 3 ? lo - hi : 0.0;
          }
        }
        double w0[3][4], wE[3][4], wO[3][4];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int r = 0; r < 4; ++r) w0[c][r] = wE[c][r] = wO[c][r] = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          mma(w0[c], dx[c][0][0], dx[c][0][1], FB[0]);   // (Dx, By)
          mma(wE[c], bp[c][0], bp[c][1], FEf);           // (Bx, By) | (Bx, Dy), even part
          mma(w0[c], dx[c][1][0], dx[c][1][1], FB[1]);
          mma(wO[c], bm[c][0], bm[c][1], FOf);           // odd part
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double* o0 = U2 + c * U2_C;
          *reinterpret_cast<double2*>(o0 + yfs[0]) = make_double2(w0[c][0], w0[c][1]);
          if (row1) *reinterpret_cast<double2*>(o0 + yfs[1]) = make_double2(w0[c][2], w0[c][3]);
          // columns 2t, 2t+1: t < 2 -> By pairs (w2 = (Bx, By)), t >= 2 -> Dy pairs (w1 = (Bx, Dy))
          const int tab = t >> 1;
          double* ob = U2 + c * U2_C + (tab == 0 ? 2 : 1) * U2_W;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == 1 && !row1) continue;
#pragma unroll
            for (int uu = 0; uu < 2; ++uu) {
              const int a = 2 * (t & 1) + uu;
              const double E = wE[c][2 * h + uu], O = wO[c][2 * h + uu];
              ob[u2o(kr[h], gl, a)] = E + O;
              ob[u2o(kr[h], gl, 7 - a)] = tab == 0 ? E - O : O - E;
            }
          }
        }
      }
      __syncwarp();

      // ---------------- fused z stage, one 8-row half (a1l = h) at a time ---------------
      // ZF: rows phi = g -> (a1l = h, a2 = g); cols a3 = 2t, 2t+1  -> gradients G[c][d][2]
      // pointwise on the two points (a1l = h, a2 = g, a3 = 2t + u), qdata r = 2h + u
      // ZB: K position (ks, t) <-> a3 = 2t + ks, A operand straight from G; rows -> U2 rows
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double G[3][3][2];
        {
          double zi[3][3][2];  // [c][w][ks]
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int w = 0; w < 3; ++w)
#pragma unroll
              for (int ks = 0; ks < 2; ++ks) zi[c][w][ks] = U2[c * U2_C + w * U2_W + zfl[ks][h]];
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int w = 0; w < 3; ++w) G[c][w][0] = G[c][w][1] = 0.0;
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
              for (int w = 0; w < 3; ++w) mma8(G[c][w], zi[c][w][ks], w == 2 ? FD[ks] : FB[ks]);
        }
        double An[2][9];   // qdata of the other half, requested now (consumed next iteration)
        if (h == 0) {
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int f = 0; f < 9; ++f) An[r][f] = __ldg(qs + ((2 + r) * 9 + f) * 32);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          double Gp[3][3];
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int d = 0; d < 3; ++d) Gp[c][d] = G[c][d][u];
          pointwise(Gp, Aq[u], re);
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int d = 0; d < 3; ++d) G[c][d][u] = Gp[c][d];
        }
        if (h == 0) {
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int f = 0; f < 9; ++f) Aq[r][f] = An[r][f];
        }
        __syncwarp();  // every lane has read its ZF inputs of rows h before they are overwritten
        double v[3][3][2];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int d = 0; d < 3; ++d) v[c][d][0] = v[c][d][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int d = 0; d < 3; ++d) mma8(v[c][d], G[c][d][ks], d == 2 ? BDp[ks] : BBp[ks]);
        // rows (a1l = h, a2 = g), cols k = 2t, 2t+1
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            double* ob = U2 + c * U2_C + d * U2_W;
            ob[zbs[0][h]] = v[c][d][0];
            if (t < 3) ob[zbs[1][h]] = v[c][d][1];
          }
      }
      __syncwarp();

      // ---------------- YB: transposed y -> T0, T1 into UX (this slice's a1 columns) ------
      {
        double vi[3][3][2][2];  // [c][d][ks][h]
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int d = 0; d < 3; ++d)
#pragma unroll
            for (int ks = 0; ks < 2; ++ks)
#pragma unroll
              for (int h = 0; h < 2; ++h) vi[c][d][ks][h] = U2[c * U2_C + d * U2_W + ybl[ks][h]];
        double t0[3][4], t1[3][4];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int r = 0; r < 4; ++r) t0[c][r] = t1[c][r] = 0.0;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            mma(t0[c], vi[c][0][ks][0], vi[c][0][ks][1], BB[ks]);   // By^T V0
            mma(t1[c], vi[c][1][ks][0], vi[c][1][ks][1], BD[ks]);   // Dy^T V1
          }
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
          for (int c = 0; c < 3; ++c) mma(t1[c], vi[c][2][ks][0], vi[c][2][ks][1], BB[ks]);  // + By^T V2
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double* ob = UX + c * UX_C + xyb;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == 0 || row1) {
              ob[ybs[0][h]] = t0[c][2 * h];
              ob[UX_V + ybs[0][h]] = t1[c][2 * h];
              if (t < 3) {
                ob[ybs[1][h]] = t0[c][2 * h + 1];
                ob[UX_V + ybs[1][h]] = t1[c][2 * h + 1];
              }
            }
          }
        }
      }
      __syncwarp();
    }
    pair_sync(el);

    // ---------------- XB: transposed x + scatter-add (tiles T = half, half+2, ...) ---------
#pragma unroll
    for (int u = 0; u < XT_PER_WARP; ++u) {
      if (WPE * u + half >= XTILES) break;
      int cc[2], jj[2], kk[2];
      bool okr[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int f = 16 * (WPE * u + half) + g + 8 * h;
        okr[h] = f < 3 * N * N;
        fibre(f, cc[h], jj[h], kk[h]);
      }
      double o[4] = {0, 0, 0, 0};
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int a1 = 4 * ks + t;
        const double* r0 = UX + cc[0] * UX_C + uxo(kk[0], jj[0], a1);
        const double* r1 = UX + cc[1] * UX_C + uxo(kk[1], jj[1], a1);
        mma(o, r0[0], r1[0], BD[ks]);         // Dx^T T0
        mma(o, r0[UX_V], r1[UX_V], BB[ks]);   // Bx^T T1
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!okr[h]) continue;
        double* dst = y + cc[h] * s.nodes + ebase + (int64_t)s.Nx * jj[h] + plane * kk[h];
#pragma unroll
        for (int uu = 0; uu < 2; ++uu) {
          const int i = 2 * t + uu;
          if (i >= N) continue;
          if (bc && cons(I0 + i, J0 + jj[h], K0 + kk[h], s)) continue;
          ELAS_DCHECK(dst >= y && (dst - y) + i < 3 * s.nodes);
          atomicAdd(dst + i, o[2 * h + uu]);
        }
      }
    }
  }
}

}  // namespace tc
}  // namespace elas
