// The fused sm_100a apply kernel: y += G^T B^T D B G x for a block of elements per CTA.
//
// One element-centric pass (macro-kernel fusion, Alg. 2): the E-vector
// gather, the forward sum factorisation (three staged 1D contractions),
// the pointwise Voigt-symmetric stress at every quadrature point, the
// transposed contractions and the scatter-add all happen inside this kernel; intermediates
// live in shared memory and registers only.  "Fibers to slices" becomes:
// every stage is a set of independent 1D fibers, one thread per fiber and the three
// displacement components blocked in registers, with shared-memory transposes between
// stages laid out so that warp accesses are bank-conflict free.
//
// Stage order per CTA (EB elements, NT threads, 4 barriers):
//   Z : gather x (zeroing Dirichlet dofs) along z-columns and contract in z with B and D
//         u[c][k]            -> Zb[c][a3], Zd[c][a3]                       (registers -> smem sZ)
//   Y : contract in y        -> Y0 = By Zb, Y1 = Dy Zb, Y2 = By Zd          (sZ -> sY)
//   X : contract in x        -> G[c][d][a1] = d u_c / d xi_d at the q points of the x-line,
//       pointwise            -> F = sigma~ A~^T (qdata A~ = sqrt(mu W) J^{-1}, r = lam/mu),
//       transposed x         -> V[c][d][i]                                  (sY -> regs -> sY)
//   Yt: transposed y         -> Wb = By^T V0 + Dy^T V1, Wd = By^T V2        (sY -> sZ)
//   Zt: transposed z + scatter: y[node] += Bz^T Wb + Dz^T Wd  (red.global.add.f64; skips
//       Dirichlet rows, whose values the init kernel already set to x)
//
// Coefficients of B, D are broadcast from shared memory into REGISTERS: on B200 a DFMA
// with a constant/uniform-register operand runs at ~20 TF/s against ~34 TF/s with all
// register operands (tools/microbench); each coefficient feeds 3
// (or 6) FMAs, one per displacement component.
#pragma once
#include "elas_internal.h"

namespace elas {

// ---------------------------------------------------------------------------------------
// compile-time layout search: minimise 128-byte wavefronts of 64-bit shared accesses
// (half-warp of 16 lanes, bank = double word mod 16, equal addresses broadcast)
// ---------------------------------------------------------------------------------------
// G = lanes per 128-byte wavefront = number of word-banks: 16 for 8-byte words, 32 for 4-byte
constexpr int halfwarp_cost(const int* addr, int n, int G = 16) {
  int total = 0;
  for (int h = 0; h < n; h += G) {
    int cnt[32] = {0};
    int worst = 0;
    for (int l = h; l < h + G && l < n; ++l) {
      bool dup = false;
      for (int m = h; m < l; ++m)
        if (addr[m] == addr[l]) dup = true;
      if (dup) continue;
      int b = ((addr[l] % G) + G) % G;
      cnt[b] += 1;
      if (cnt[b] > worst) worst = cnt[b];
    }
    total += worst;
  }
  return total;
}

// a3-stride of the Z buffer: stage Y/Yt lanes are (i fast, a3 slow)
constexpr int pick_SA(int N, int Q, int G = 16) {
  int best = N * N, best_cost = 1 << 30;
  for (int SA = N * N; SA < N * N + G; ++SA) {
    int addr[512] = {0};
    int n = 0;
    for (int a3 = 0; a3 < Q; ++a3)
      for (int i = 0; i < N; ++i) addr[n++] = a3 * SA + i;
    int c = halfwarp_cost(addr, n, G);
    if (c < best_cost) { best_cost = c; best = SA; }
  }
  return best;
}

// a2-stride of the Y buffer: stage X lanes are lines L = a3 + Q a2 (a3 fast), a3-stride LN
constexpr int pick_S2(int N, int Q, int LN, int G = 16) {
  int best = Q * LN, best_cost = 1 << 30;
  for (int S2 = Q * LN; S2 < Q * LN + G; ++S2) {
    int addr[512] = {0};
    int n = 0;
    for (int a2 = 0; a2 < Q; ++a2)
      for (int a3 = 0; a3 < Q; ++a3) addr[n++] = a2 * S2 + a3 * LN;
    int c = halfwarp_cost(addr, n, G);
    if (c < best_cost) { best_cost = c; best = S2; }
  }
  return best;
}

// a3-stride (line stride) of the Y buffer.  Stage X reads and writes whole x-lines, one lane per
// line (a3 fast), so an even node count N as the stride puts the lanes of a half-warp on few
// banks: at p = 7 (N = 8) 9 lanes share 2 double-word banks and 76 % of that stage's shared
// wavefronts are conflicts (ncu, round 2; tools/smem_by_line.py).  LNO: the next odd stride
// instead (stage Y/Yt then pay a 2-way conflict on one bank per half-warp).
constexpr int pick_LN(int N, int LNO) { return LNO ? (N | 1) : N; }

// element strides of the Z and Y buffers: at low order one warp spans several elements, so
// pad the element strides to minimise conflicts over whole warps of every stage's pattern
constexpr int elem_pattern_cost(int N, int Q, int SA, int S2, int LN, int ZE, int YE, int NT, int G = 16) {
  int total = 0;
  int addr[512] = {0};
  const int lanes = NT < 512 ? NT : 512;
  // stage Z / Zt: Z buffer, lanes (i, j, el)
  for (int w = 0; w < lanes; ++w) addr[w] = (w / (N * N)) * ZE + ((w / N) % N) * N + w % N;
  total += halfwarp_cost(addr, lanes, G);
  // stage Y / Yt: Z buffer and Y buffer, lanes (i, a3, el)
  for (int w = 0; w < lanes; ++w) addr[w] = (w / (N * Q)) * ZE + ((w / N) % Q) * SA + w % N;
  total += halfwarp_cost(addr, lanes, G);
  for (int w = 0; w < lanes; ++w) addr[w] = (w / (N * Q)) * YE + ((w / N) % Q) * LN + w % N;
  total += halfwarp_cost(addr, lanes, G);
  // stage X: Y buffer, lanes (a3, a2, el)
  for (int w = 0; w < lanes; ++w) addr[w] = (w / (Q * Q)) * YE + ((w / Q) % Q) * S2 + (w % Q) * LN;
  total += halfwarp_cost(addr, lanes, G);
  return total;
}

constexpr int pick_ZE(int N, int Q, int SA, int S2, int LN, int ZE0, int YE0, int NT, int G = 16) {
  int best = ZE0, bc = 1 << 30;
  for (int p = 0; p < G; ++p) {
    const int c = elem_pattern_cost(N, Q, SA, S2, LN, ZE0 + p, YE0, NT, G);
    if (c < bc) { bc = c; best = ZE0 + p; }
  }
  return best;
}

constexpr int pick_YE(int N, int Q, int SA, int S2, int LN, int ZE, int YE0, int NT, int G = 16) {
  int best = YE0, bc = 1 << 30;
  for (int p = 0; p < G; ++p) {
    const int c = elem_pattern_cost(N, Q, SA, S2, LN, ZE, YE0 + p, NT, G);
    if (c < bc) { bc = c; best = YE0 + p; }
  }
  return best;
}

constexpr int kSmemLimit = 227 * 1024;
#ifndef ELAS_EB_BY_COLUMNS
#define ELAS_EB_BY_COLUMNS 0
#endif
#ifndef ELAS_QD_STAGING
#define ELAS_QD_STAGING 1
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
#ifndef ELAS_L2_PREFETCH
#define ELAS_L2_PREFETCH 1
#endif

#ifndef ELAS_NT
#define ELAS_NT 128
#endif

// WB: bytes per stored word (8: FP64 kernels; 4: the FP32 folded kernel).  All counts below
// are in words of that size.
constexpr int qd_stride_words(int q, int WB) { return WB == 8 ? (9 * q * q * q + 1) & ~1 : (9 * q * q * q + 3) & ~3; }

// PAD = 0: unpadded tiles (minimal shared memory, bank conflicts accepted)
template <int P, int Q, int TABSZ = 2 * Q * (P + 1), int NTHR = ELAS_NT, int WB = 8, int PAD = 1, int LNO = 0>
struct Cfg {
  static constexpr int N = P + 1;
  static constexpr int NT = NTHR;
  static constexpr int G = 128 / WB;       // word-banks per wavefront
  static constexpr int AL = 16 / WB;       // words per 16 bytes
  static constexpr int SA = PAD ? pick_SA(N, Q, G) : N * N;
  static constexpr int ZV = Q * SA;        // variant stride (Zb | Zd)
  static constexpr int ZC = 2 * ZV;        // component stride
  static constexpr int LN = pick_LN(N, LNO);  // a3-stride (x-line) of the Y buffer
  static constexpr int S2 = PAD ? pick_S2(N, Q, LN, G) : Q * LN;
  static constexpr int ZE = PAD ? pick_ZE(N, Q, SA, S2, LN, 3 * ZC, 9 * Q * S2, NT, G) : 3 * ZC;  // element stride
  static constexpr int YV = Q * S2;        // variant stride (Y0 | Y1 | Y2)
  static constexpr int YC = 3 * YV;        // component stride
  static constexpr int YE = PAD ? pick_YE(N, Q, SA, S2, LN, ZE, 3 * YC, NT, G) : 3 * YC;  // element stride
  static constexpr int TAB = (TABSZ + AL - 1) & ~(AL - 1);  // coefficient tables (B then D, or folded)
  // elements per CTA: enough x-lines for every thread in stage X; at low order also enough
  // z-columns (N^2 per element) to keep every thread busy in stages Z and Zt.
  static constexpr int EB_lines = (NT / (Q * Q)) > 0 ? NT / (Q * Q) : 1;
  static constexpr int EB_cols = (NT + N * N - 1) / (N * N);
  static constexpr int EB_threads = (ELAS_EB_BY_COLUMNS && EB_cols > EB_lines) ? EB_cols : EB_lines;
  static constexpr int EB_smem = (kSmemLimit / WB - TAB) / (ZE + YE);
  static constexpr int EB = EB_threads < EB_smem ? EB_threads : EB_smem;
  static constexpr int QDE = qd_stride_words(Q, WB);           // qdata words per element
  static constexpr int BASE = (TAB + EB * (ZE + YE) + AL - 1) & ~(AL - 1);  // 16-B aligned start of sQ
  // Stage the CTA's quadrature data into shared memory with one TMA bulk copy when two CTAs
  // per SM still fit (latency of the qdata stream then overlaps stages Z and Y).
  static constexpr bool STAGE_QD = ELAS_QD_STAGING && (size_t)WB * (size_t)(BASE + EB * QDE) + 16 <= (size_t)kSmemLimit / 2;
  static constexpr size_t smem = STAGE_QD ? (size_t)WB * (size_t)(BASE + EB * QDE) + 16 : (size_t)WB * (size_t)(TAB + EB * (ZE + YE));
  static_assert(EB >= 1, "element does not fit in shared memory");
};

__device__ __forceinline__ bool is_constrained(int I, int J, int K, const Slab& s) {
  const uint32_t f = s.faces;
  return ((f & ELAS_FACE_XMIN) && I == 0) || ((f & ELAS_FACE_XMAX) && I == s.Nx - 1) ||
         ((f & ELAS_FACE_YMIN) && J == 0) || ((f & ELAS_FACE_YMAX) && J == s.Ny - 1) ||
         ((f & ELAS_FACE_ZMIN) && K == 0) || ((f & ELAS_FACE_ZMAX) && K == s.Nz - 1);
}

// sigma~ = r tr(H) I + H + H^T with H = G A~ ; F = sigma~ A~^T   (Voigt-symmetric: 6 unique)
__device__ __forceinline__ void pointwise(double (&g)[3][3], const double (&A)[9], double r) {
  double H[3][3];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int m = 0; m < 3; ++m) H[c][m] = fma(g[c][2], A[6 + m], fma(g[c][1], A[3 + m], g[c][0] * A[m]));
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
      g[c][d] = fma(S[c][2], A[3 * d + 2], fma(S[c][1], A[3 * d + 1], S[c][0] * A[3 * d]));
}

// CTAs per SM the register allocation targets (ELAS_MINB_P<p>, default 1 = up to 255 regs)
#ifndef ELAS_MINB_P4
#define ELAS_MINB_P4 3   // measured: p = 4 at 3 CTAs/SM (168 regs) 20.8 -> 21.3 GDoF/s
#endif
#ifndef ELAS_MINB_DEFAULT
#define ELAS_MINB_DEFAULT 1
#endif
template <int P> struct MinBlocks { static constexpr int value = ELAS_MINB_DEFAULT; };
#ifdef ELAS_MINB_P2
template <> struct MinBlocks<2> { static constexpr int value = ELAS_MINB_P2; };
#endif
#ifdef ELAS_MINB_P3
template <> struct MinBlocks<3> { static constexpr int value = ELAS_MINB_P3; };
#endif
#ifdef ELAS_MINB_P4
template <> struct MinBlocks<4> { static constexpr int value = ELAS_MINB_P4; };
#endif
#ifdef ELAS_MINB_P5
template <> struct MinBlocks<5> { static constexpr int value = ELAS_MINB_P5; };
#endif

template <int P, int Q>
__global__ void __launch_bounds__(Cfg<P, Q>::NT, MinBlocks<P>::value)
    apply_kernel(const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ qd,
                 const double* __restrict__ rr, const double* __restrict__ tables, Slab s,
                 int64_t e_begin, int64_t e_end, int pref_ctas) {
  using C = Cfg<P, Q>;
  constexpr int N = C::N;
  constexpr int NT = C::NT;
  constexpr int EB = C::EB;
  extern __shared__ double smem[];
  double* sB = smem;            // B[a][i] = l_i(g_a), Q x N
  double* sD = smem + Q * N;    // D[a][i] = l_i'(g_a)
  double* sZ = smem + C::TAB;
  double* sY = sZ + EB * C::ZE;
  double* sQ = smem + C::BASE;                                      // staged qdata (STAGE_QD)
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + C::BASE + EB * C::QDE);

  const int tid = threadIdx.x;
  const int64_t e0 = e_begin + (int64_t)blockIdx.x * EB;
  const int ne = (int)((e_end - e0) < EB ? (e_end - e0) : EB);
  if constexpr (C::STAGE_QD) {
    if (tid == 0) {
      const uint32_t bar = smem_u32(mbar);
      const uint32_t bytes = (uint32_t)(8 * ne * C::QDE);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sQ)),
          "l"(qd + e0 * (int64_t)C::QDE), "r"(bytes), "r"(bar)
          : "memory");
    }
  }
  for (int t = tid; t < C::TAB; t += NT) sB[t] = tables[t];
  const int64_t plane = (int64_t)s.Nx * s.Ny;
#if ELAS_L2_PREFETCH
  // Pull the quadrature data of the batch that will run one wave later into L2 (TMA bulk
  // prefetch: no registers or shared memory), so stage X hits L2 instead of HBM.
  if (tid == 0 && pref_ctas > 0) {
    const int64_t pe0 = e0 + (int64_t)pref_ctas * EB;
    if (pe0 < e_end) {
      const int64_t pne = (e_end - pe0) < EB ? (e_end - pe0) : EB;
      const uintptr_t a0 = (uintptr_t)(qd + pe0 * (int64_t)C::QDE);
      const uintptr_t a1 = a0 + (uintptr_t)(pne * C::QDE * 8);
      const uintptr_t lo = a0 & ~(uintptr_t)15, hi = (a1 + 15) & ~(uintptr_t)15;  // 16-B granules
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((uint32_t)(hi - lo)) : "memory");
    }
  }
#endif
  const bool bc = s.faces != 0;
  __syncthreads();

  // ---------------- Stage Z: gather + contraction in z --------------------------------
  for (int w = tid; w < ne * N * N; w += NT) {
    const int i = w % N, j = (w / N) % N, el = w / (N * N);
    const int64_t e = e0 + el;
    const int ex = (int)(e % s.nx), ey = (int)((e / s.nx) % s.ny), ez = (int)(e / ((int64_t)s.nx * s.ny));
    const int I = ex * P + i, J = ey * P + j;
    const int64_t base = I + (int64_t)s.Nx * J + plane * ((int64_t)ez * P);
    double u[3][N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const bool cons = bc && is_constrained(I, J, ez * P + k, s);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        ELAS_DCHECK(base >= 0 && c * s.nodes + base + k * plane < 3 * s.nodes);
        u[c][k] = cons ? 0.0 : __ldg(x + c * s.nodes + base + k * plane);
      }
    }
    double* dst = sZ + el * C::ZE + j * N + i;
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      double zb[3] = {0.0, 0.0, 0.0}, zd[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double b = sB[a * N + k], d = sD[a * N + k];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          zb[c] = fma(b, u[c][k], zb[c]);
          zd[c] = fma(d, u[c][k], zd[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        dst[c * C::ZC + a * C::SA] = zb[c];
        dst[c * C::ZC + C::ZV + a * C::SA] = zd[c];
      }
    }
  }
  __syncthreads();

  // ---------------- Stage Y: contraction in y ------------------------------------------
  for (int w = tid; w < ne * Q * N; w += NT) {
    const int i = w % N, a3 = (w / N) % Q, el = w / (N * Q);
    const double* src = sZ + el * C::ZE + a3 * C::SA + i;
    double zb[3][N], zd[3][N];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < N; ++j) {
        zb[c][j] = src[c * C::ZC + j * N];
        zd[c][j] = src[c * C::ZC + C::ZV + j * N];
      }
    double* dst = sY + el * C::YE + a3 * C::LN + i;
#pragma unroll
    for (int a2 = 0; a2 < Q; ++a2) {
      double y0[3] = {0, 0, 0}, y1[3] = {0, 0, 0}, y2[3] = {0, 0, 0};
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const double b = sB[a2 * N + j], d = sD[a2 * N + j];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          y0[c] = fma(b, zb[c][j], y0[c]);
          y1[c] = fma(d, zb[c][j], y1[c]);
          y2[c] = fma(b, zd[c][j], y2[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        dst[c * C::YC + a2 * C::S2] = y0[c];
        dst[c * C::YC + C::YV + a2 * C::S2] = y1[c];
        dst[c * C::YC + 2 * C::YV + a2 * C::S2] = y2[c];
      }
    }
  }
  __syncthreads();

  // ---------------- Stage X + pointwise + transposed X ---------------------------------
  if constexpr (C::STAGE_QD) {
    const uint32_t bar = smem_u32(mbar);
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(bar)
        : "memory");
  }
  for (int w = tid; w < ne * Q * Q; w += NT) {
    const int L = w % (Q * Q), el = w / (Q * Q);
    const int a3 = L % Q, a2 = L / Q;
    const int64_t e = e0 + el;
    double* line = sY + el * C::YE + a2 * C::S2 + a3 * C::LN;
    double g[3][3][Q];
#pragma unroll
    for (int v = 0; v < 3; ++v) {
      const double* tab = (v == 0) ? sD : sB;
      double f[3][N];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int i = 0; i < N; ++i) f[c][i] = line[c * C::YC + v * C::YV + i];
#pragma unroll
      for (int a1 = 0; a1 < Q; ++a1) {
        double acc[3] = {0, 0, 0};
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const double t = tab[a1 * N + i];
#pragma unroll
          for (int c = 0; c < 3; ++c) acc[c] = fma(t, f[c][i], acc[c]);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) g[c][v][a1] = acc[c];
      }
    }
    const double r = __ldg(rr + e);
    const double* qp = C::STAGE_QD ? sQ + el * C::QDE + L : qd + e * (int64_t)C::QDE + L;
    double An[9];
#pragma unroll
    for (int f = 0; f < 9; ++f) An[f] = qp[f * Q * Q];
#pragma unroll
    for (int a1 = 0; a1 < Q; ++a1) {
      double A[9];
#pragma unroll
      for (int f = 0; f < 9; ++f) A[f] = An[f];
      if (a1 + 1 < Q) {
#pragma unroll
        for (int f = 0; f < 9; ++f) An[f] = qp[((a1 + 1) * 9 + f) * Q * Q];
      }
      double G[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) G[c][d] = g[c][d][a1];
      pointwise(G, A, r);
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) g[c][d][a1] = G[c][d];
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double* tab = (d == 0) ? sD : sB;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double acc[3] = {0, 0, 0};
#pragma unroll
        for (int a1 = 0; a1 < Q; ++a1) {
          const double t = tab[a1 * N + i];
#pragma unroll
          for (int c = 0; c < 3; ++c) acc[c] = fma(t, g[c][d][a1], acc[c]);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) line[c * C::YC + d * C::YV + i] = acc[c];
      }
    }
  }
  __syncthreads();

  // ---------------- Stage Yt: transposed contraction in y ------------------------------
  for (int w = tid; w < ne * Q * N; w += NT) {
    const int i = w % N, a3 = (w / N) % Q, el = w / (N * Q);
    const double* src = sY + el * C::YE + a3 * C::LN + i;
    double wb[3][N], wd[3][N];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < N; ++j) wb[c][j] = wd[c][j] = 0.0;
#pragma unroll
    for (int a2 = 0; a2 < Q; ++a2) {
      double v0[3], v1[3], v2[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        v0[c] = src[c * C::YC + a2 * C::S2];
        v1[c] = src[c * C::YC + C::YV + a2 * C::S2];
        v2[c] = src[c * C::YC + 2 * C::YV + a2 * C::S2];
      }
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const double b = sB[a2 * N + j], d = sD[a2 * N + j];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          wb[c][j] = fma(d, v1[c], fma(b, v0[c], wb[c][j]));
          wd[c][j] = fma(b, v2[c], wd[c][j]);
        }
      }
    }
    double* dst = sZ + el * C::ZE + a3 * C::SA + i;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < N; ++j) {
        dst[c * C::ZC + j * N] = wb[c][j];
        dst[c * C::ZC + C::ZV + j * N] = wd[c][j];
      }
  }
  __syncthreads();

  // ---------------- Stage Zt: transposed contraction in z + scatter-add ----------------
  for (int w = tid; w < ne * N * N; w += NT) {
    const int i = w % N, j = (w / N) % N, el = w / (N * N);
    const int64_t e = e0 + el;
    const int ex = (int)(e % s.nx), ey = (int)((e / s.nx) % s.ny), ez = (int)(e / ((int64_t)s.nx * s.ny));
    const double* src = sZ + el * C::ZE + j * N + i;
    double o[3][N];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int k = 0; k < N; ++k) o[c][k] = 0.0;
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      double wb[3], wd[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        wb[c] = src[c * C::ZC + a * C::SA];
        wd[c] = src[c * C::ZC + C::ZV + a * C::SA];
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double b = sB[a * N + k], d = sD[a * N + k];
#pragma unroll
        for (int c = 0; c < 3; ++c) o[c][k] = fma(d, wd[c], fma(b, wb[c], o[c][k]));
      }
    }
    const int I = ex * P + i, J = ey * P + j;
    const int64_t base = I + (int64_t)s.Nx * J + plane * ((int64_t)ez * P);
#pragma unroll
    for (int k = 0; k < N; ++k) {
      if (bc && is_constrained(I, J, ez * P + k, s)) continue;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        ELAS_DCHECK(base >= 0 && c * s.nodes + base + k * plane < 3 * s.nodes);
        atomicAdd(y + c * s.nodes + base + k * plane, o[c][k]);
      }
    }
  }
}

template <int P, int Q>
cudaError_t launch_apply_pq(const Slab& s, const double* x, double* y, const double* qd,
                            const double* rr, const double* tables, int64_t e_begin, int64_t e_end,
                            cudaStream_t st) {
  using C = Cfg<P, Q>;
  static KernelPrep prep;   // per device
  int pref = 0;
  cudaError_t err = prep.prep(apply_kernel<P, Q>, C::NT, C::smem, &pref);
  if (err != cudaSuccess) return err;
  const int64_t ne = e_end - e_begin;
  if (ne <= 0) return cudaSuccess;
  const int64_t grid = (ne + C::EB - 1) / C::EB;
  apply_kernel<P, Q><<<(unsigned)grid, C::NT, C::smem, st>>>(x, y, qd, rr, tables, s, e_begin, e_end, pref);
  return cudaGetLastError();
}

template <int P, int Q>
void info_pq(ApplyLaunch* info) {
  using C = Cfg<P, Q>;
  info->threads = C::NT;
  info->elems_per_cta = C::EB;
  info->smem_bytes = C::smem;
}

}  // namespace elas

// Instantiate the two quadrature variants q = p+1, p+2 of one degree P.
#define ELAS_DEFINE_DEGREE(P)                                                                   \
  ELAS_DCHECK_READER(dcheck_simt_p##P)                                                          \
  namespace elas {                                                                              \
  cudaError_t apply_info_p##P(int q, ApplyLaunch* info) {                                       \
    if (q == P + 1) info_pq<P, P + 1>(info);                                                    \
    else if (q == P + 2) info_pq<P, P + 2>(info);                                               \
    else return cudaErrorInvalidValue;                                                          \
    return cudaSuccess;                                                                         \
  }                                                                                             \
  cudaError_t apply_launch_p##P(int q, const Slab& s, const double* x, double* y,               \
                                const double* qd, const double* rr, const double* tables,       \
                                int64_t e_begin, int64_t e_end, cudaStream_t st) {              \
    if (q == P + 1) return launch_apply_pq<P, P + 1>(s, x, y, qd, rr, tables, e_begin, e_end, st); \
    if (q == P + 2) return launch_apply_pq<P, P + 2>(s, x, y, qd, rr, tables, e_begin, e_end, st); \
    return cudaErrorInvalidValue;                                                               \
  }                                                                                             \
  }
