// Even-odd folded variant of the fused SIMT apply kernel (ELAS_VARIANT_FOLDED).
//
// Same element pass, stage order, shared-memory tiles, qdata layout and scatter as
// elas_apply.cuh (gather -> Z -> Y -> X + pointwise + Xt -> Yt -> Zt + scatter-add); only the
// 1D contractions change.  GLL nodes and Gauss points are symmetric about 1/2, so
// B[q-1-a][n-1-i] = B[a][i] and D[q-1-a][n-1-i] = -D[a][i].  Folding the input of every
// contraction into its even and odd halves,
//   u+_i = u_i + u_{n-1-i},  u-_i = u_i - u_{n-1-i}   (i < n/2; u_mid alone when n is odd)
// gives each PAIR of outputs (a, q-1-a) from one even and one odd half-length dot product:
//   E = sum FE[a][i] u+_i,  O = sum FO[a][i] u-_i,   out_a = E + O,  out_{q-1-a} = s (E - O).
// That halves the FMAs of the sum factorisation (Eq. 6's B_1D/D_1D factors) and
// the coefficient loads from shared memory; the algorithmic flop count the bench reports
// is unchanged, so a folded kernel's roofline fraction counts the plain
// sum-factorisation work it replaces.  Folded tables: elas_tables.cpp host_fold_table.
//
// The transposed contractions accumulate, per pair of points (a, q-1-a), into two sums per
// output pair of nodes, X and Y, so that out_j = X + Y and out_{n-1-j} = X - Y:
//   B-part: X += BE_B v+,  Y += BO_B v-;   D-part (parity -1): X += BO_D w-,  Y += BE_D w+.
#pragma once
#include "elas_apply.cuh"

namespace elas {

template <int P, int Q>
struct Fold {
  static constexpr int N = P + 1;
  static constexpr int NE = (N + 1) / 2, NH = N / 2, QE = (Q + 1) / 2, QH = Q / 2;
  static constexpr int FE = 0, FO = QE * NE, BE = QE * N, BO = QE * N + NE * QE;
  static constexpr int TS = QE * N + NE * Q;   // doubles per folded table (== fold_table_size)
  static constexpr int NHX = NH > 0 ? NH : 1;
  static constexpr int QHX = QH > 0 ? QH : 1;
};

template <int P, int Q>
using CfgEO = Cfg<P, Q, 2 * Fold<P, Q>::TS>;

// u (n values per component) -> even (ne) / odd (nh) halves
template <int N, int NE, int NHX>
__device__ __forceinline__ void fold_in(const double (&u)[3][N], double (&up)[3][NE], double (&um)[3][NHX]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      up[c][i] = u[c][i] + u[c][N - 1 - i];
      um[c][i] = u[c][i] - u[c][N - 1 - i];
    }
    if (N & 1) up[c][N / 2] = u[c][N / 2];
  }
}

template <int P, int Q>
__global__ void __launch_bounds__(CfgEO<P, Q>::NT, MinBlocks<P>::value)
    apply_eo_kernel(const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ qd,
                    const double* __restrict__ rr, const double* __restrict__ tables, Slab s,
                    int64_t e_begin, int64_t e_end, int pref_ctas) {
  using C = CfgEO<P, Q>;
  using F = Fold<P, Q>;
  constexpr int N = C::N, NT = C::NT, EB = C::EB;
  constexpr int NE = F::NE, NH = F::NH, QE = F::QE, QH = F::QH, NHX = F::NHX;
  extern __shared__ double smem[];
  double* tB = smem;            // folded B (parity +1)
  double* tD = smem + F::TS;    // folded D (parity -1)
  double* sZ = smem + C::TAB;
  double* sY = sZ + EB * C::ZE;
  double* sQ = smem + C::BASE;
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
  {
    const double* ft = tables + 2 * Q * N;   // fold(B) | fold(D) follow the plain tables
    for (int t = tid; t < 2 * F::TS; t += NT) smem[t] = ft[t];
  }
  const int64_t plane = (int64_t)s.Nx * s.Ny;
#if ELAS_L2_PREFETCH
  if (tid == 0 && pref_ctas > 0) {
    const int64_t pe0 = e0 + (int64_t)pref_ctas * EB;
    if (pe0 < e_end) {
      const int64_t pne = (e_end - pe0) < EB ? (e_end - pe0) : EB;
      const uintptr_t a0 = (uintptr_t)(qd + pe0 * (int64_t)C::QDE);
      const uintptr_t a1 = a0 + (uintptr_t)(pne * C::QDE * 8);
      const uintptr_t lo = a0 & ~(uintptr_t)15, hi = (a1 + 15) & ~(uintptr_t)15;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((uint32_t)(hi - lo)) : "memory");
    }
  }
#endif
  const bool bc = s.faces != 0;
  __syncthreads();

  // ---------------- Stage Z: gather + folded contraction in z ---------------------------
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
      for (int c = 0; c < 3; ++c) u[c][k] = cons ? 0.0 : __ldg(x + c * s.nodes + base + k * plane);
    }
    double up[3][NE], um[3][NHX];
    fold_in<N, NE, NHX>(u, up, um);
    double* dst = sZ + el * C::ZE + j * N + i;
#pragma unroll
    for (int a = 0; a < QE; ++a) {
      const bool mid = (Q & 1) && a == QH;
      double eb[3] = {0, 0, 0}, ob[3] = {0, 0, 0}, ed[3] = {0, 0, 0}, od[3] = {0, 0, 0};
#pragma unroll
      for (int k = 0; k < NE; ++k) {
        const double b = tB[F::FE + a * NE + k];
#pragma unroll
        for (int c = 0; c < 3; ++c) eb[c] = fma(b, up[c][k], eb[c]);
        if (!mid) {
          const double d = tD[F::FE + a * NE + k];
#pragma unroll
          for (int c = 0; c < 3; ++c) ed[c] = fma(d, up[c][k], ed[c]);
        }
      }
#pragma unroll
      for (int k = 0; k < NH; ++k) {
        const double d = tD[F::FO + a * NH + k];
#pragma unroll
        for (int c = 0; c < 3; ++c) od[c] = fma(d, um[c][k], od[c]);
        if (!mid) {
          const double b = tB[F::FO + a * NH + k];
#pragma unroll
          for (int c = 0; c < 3; ++c) ob[c] = fma(b, um[c][k], ob[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        dst[c * C::ZC + a * C::SA] = eb[c] + ob[c];
        dst[c * C::ZC + C::ZV + a * C::SA] = ed[c] + od[c];
        if (!mid) {
          dst[c * C::ZC + (Q - 1 - a) * C::SA] = eb[c] - ob[c];
          dst[c * C::ZC + C::ZV + (Q - 1 - a) * C::SA] = od[c] - ed[c];
        }
      }
    }
  }
  __syncthreads();

  // ---------------- Stage Y: folded contraction in y ------------------------------------
  for (int w = tid; w < ne * Q * N; w += NT) {
    const int i = w % N, a3 = (w / N) % Q, el = w / (N * Q);
    const double* src = sZ + el * C::ZE + a3 * C::SA + i;
    double bp[3][NE], bm[3][NHX], dp[3][NE], dm[3][NHX];
    {
      double zb[3][N], zd[3][N];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int j = 0; j < N; ++j) {
          zb[c][j] = src[c * C::ZC + j * N];
          zd[c][j] = src[c * C::ZC + C::ZV + j * N];
        }
      fold_in<N, NE, NHX>(zb, bp, bm);
      fold_in<N, NE, NHX>(zd, dp, dm);
    }
    double* dst = sY + el * C::YE + a3 * N + i;
#pragma unroll
    for (int a2 = 0; a2 < QE; ++a2) {
      const bool mid = (Q & 1) && a2 == QH;
      // y0 = By zb (+1), y1 = Dy zb (-1), y2 = By zd (+1)
      double e0[3] = {0, 0, 0}, o0[3] = {0, 0, 0}, e1[3] = {0, 0, 0}, o1[3] = {0, 0, 0};
      double e2[3] = {0, 0, 0}, o2[3] = {0, 0, 0};
#pragma unroll
      for (int j = 0; j < NE; ++j) {
        const double b = tB[F::FE + a2 * NE + j];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          e0[c] = fma(b, bp[c][j], e0[c]);
          e2[c] = fma(b, dp[c][j], e2[c]);
        }
        if (!mid) {
          const double d = tD[F::FE + a2 * NE + j];
#pragma unroll
          for (int c = 0; c < 3; ++c) e1[c] = fma(d, bp[c][j], e1[c]);
        }
      }
#pragma unroll
      for (int j = 0; j < NH; ++j) {
        const double d = tD[F::FO + a2 * NH + j];
#pragma unroll
        for (int c = 0; c < 3; ++c) o1[c] = fma(d, bm[c][j], o1[c]);
        if (!mid) {
          const double b = tB[F::FO + a2 * NH + j];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            o0[c] = fma(b, bm[c][j], o0[c]);
            o2[c] = fma(b, dm[c][j], o2[c]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        dst[c * C::YC + a2 * C::S2] = e0[c] + o0[c];
        dst[c * C::YC + C::YV + a2 * C::S2] = e1[c] + o1[c];
        dst[c * C::YC + 2 * C::YV + a2 * C::S2] = e2[c] + o2[c];
        if (!mid) {
          dst[c * C::YC + (Q - 1 - a2) * C::S2] = e0[c] - o0[c];
          dst[c * C::YC + C::YV + (Q - 1 - a2) * C::S2] = o1[c] - e1[c];
          dst[c * C::YC + 2 * C::YV + (Q - 1 - a2) * C::S2] = e2[c] - o2[c];
        }
      }
    }
  }
  __syncthreads();

  // ---------------- Stage X + pointwise + transposed X (folded) -------------------------
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
    double* line = sY + el * C::YE + a2 * C::S2 + a3 * N;
    double g[3][3][Q];
#pragma unroll
    for (int v = 0; v < 3; ++v) {
      const double* tab = (v == 0) ? tD : tB;   // x-derivative for v = 0 (parity -1)
      const bool odd = (v == 0);
      double fp[3][NE], fm[3][NHX];
      {
        double f[3][N];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int i = 0; i < N; ++i) f[c][i] = line[c * C::YC + v * C::YV + i];
        fold_in<N, NE, NHX>(f, fp, fm);
      }
#pragma unroll
      for (int a1 = 0; a1 < QE; ++a1) {
        const bool mid = (Q & 1) && a1 == QH;
        double ev[3] = {0, 0, 0}, ov[3] = {0, 0, 0};
        if (!(mid && odd)) {
#pragma unroll
          for (int i = 0; i < NE; ++i) {
            const double t = tab[F::FE + a1 * NE + i];
#pragma unroll
            for (int c = 0; c < 3; ++c) ev[c] = fma(t, fp[c][i], ev[c]);
          }
        }
        if (!(mid && !odd)) {
#pragma unroll
          for (int i = 0; i < NH; ++i) {
            const double t = tab[F::FO + a1 * NH + i];
#pragma unroll
            for (int c = 0; c < 3; ++c) ov[c] = fma(t, fm[c][i], ov[c]);
          }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          g[c][v][a1] = ev[c] + ov[c];
          if (!mid) g[c][v][Q - 1 - a1] = odd ? ov[c] - ev[c] : ev[c] - ov[c];
        }
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
      const double* tab = (d == 0) ? tD : tB;
      const bool odd = (d == 0);
      // fold over the points a1 in place: g[.][a] <- g_a + g_{q-1-a}, g[.][q-1-a] <- g_a - g_{q-1-a}
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int a = 0; a < QH; ++a) {
          const double lo = g[c][d][a], hi = g[c][d][Q - 1 - a];
          g[c][d][a] = lo + hi;
          g[c][d][Q - 1 - a] = lo - hi;
        }
#pragma unroll
      for (int i = 0; i < NE; ++i) {
        const bool mid = (N & 1) && i == NH;
        double ev[3] = {0, 0, 0}, ov[3] = {0, 0, 0};
        if (!(mid && odd)) {
#pragma unroll
          for (int a = 0; a < QE; ++a) {
            const double t = tab[F::BE + i * QE + a];
#pragma unroll
            for (int c = 0; c < 3; ++c) ev[c] = fma(t, g[c][d][a], ev[c]);
          }
        }
        if (!(mid && !odd)) {
#pragma unroll
          for (int a = 0; a < QH; ++a) {
            const double t = tab[F::BO + i * QH + a];
#pragma unroll
            for (int c = 0; c < 3; ++c) ov[c] = fma(t, g[c][d][Q - 1 - a], ov[c]);
          }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          line[c * C::YC + d * C::YV + i] = ev[c] + ov[c];
          if (!mid) line[c * C::YC + d * C::YV + N - 1 - i] = odd ? ov[c] - ev[c] : ev[c] - ov[c];
        }
      }
    }
  }
  __syncthreads();

  // ---------------- Stage Yt: folded transposed contraction in y ------------------------
  for (int w = tid; w < ne * Q * N; w += NT) {
    const int i = w % N, a3 = (w / N) % Q, el = w / (N * Q);
    const double* src = sY + el * C::YE + a3 * N + i;
    // wb = By^T V0 + Dy^T V1, wd = By^T V2 ; X/Y sums per node pair (j, n-1-j)
    double bX[3][NE], bY[3][NE], dX[3][NE], dY[3][NE];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < NE; ++j) bX[c][j] = bY[c][j] = dX[c][j] = dY[c][j] = 0.0;
#pragma unroll
    for (int a = 0; a < QE; ++a) {
      const bool mid = (Q & 1) && a == QH;
      double v0p[3], v0m[3], v1p[3], v1m[3], v2p[3], v2m[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double l0 = src[c * C::YC + a * C::S2];
        const double l1 = src[c * C::YC + C::YV + a * C::S2];
        const double l2 = src[c * C::YC + 2 * C::YV + a * C::S2];
        if (mid) {
          v0p[c] = l0; v1p[c] = l1; v2p[c] = l2;
          v0m[c] = v1m[c] = v2m[c] = 0.0;
        } else {
          const double h0 = src[c * C::YC + (Q - 1 - a) * C::S2];
          const double h1 = src[c * C::YC + C::YV + (Q - 1 - a) * C::S2];
          const double h2 = src[c * C::YC + 2 * C::YV + (Q - 1 - a) * C::S2];
          v0p[c] = l0 + h0; v0m[c] = l0 - h0;
          v1p[c] = l1 + h1; v1m[c] = l1 - h1;
          v2p[c] = l2 + h2; v2m[c] = l2 - h2;
        }
      }
#pragma unroll
      for (int j = 0; j < NE; ++j) {
        const bool jmid = (N & 1) && j == NH;
        const double be = tB[F::BE + j * QE + a];
        const double de = tD[F::BE + j * QE + a];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          bX[c][j] = fma(be, v0p[c], bX[c][j]);
          dX[c][j] = fma(be, v2p[c], dX[c][j]);
          if (!jmid) bY[c][j] = fma(de, v1p[c], bY[c][j]);
        }
        if (!mid) {
          const double bo = tB[F::BO + j * QH + a];
          const double dO = tD[F::BO + j * QH + a];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            bX[c][j] = fma(dO, v1m[c], bX[c][j]);
            if (!jmid) {
              bY[c][j] = fma(bo, v0m[c], bY[c][j]);
              dY[c][j] = fma(bo, v2m[c], dY[c][j]);
            }
          }
        }
      }
    }
    double* dst = sZ + el * C::ZE + a3 * C::SA + i;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < NE; ++j) {
        const bool jmid = (N & 1) && j == NH;
        dst[c * C::ZC + j * N] = jmid ? bX[c][j] : bX[c][j] + bY[c][j];
        dst[c * C::ZC + C::ZV + j * N] = jmid ? dX[c][j] : dX[c][j] + dY[c][j];
        if (!jmid) {
          dst[c * C::ZC + (N - 1 - j) * N] = bX[c][j] - bY[c][j];
          dst[c * C::ZC + C::ZV + (N - 1 - j) * N] = dX[c][j] - dY[c][j];
        }
      }
  }
  __syncthreads();

  // ---------------- Stage Zt: folded transposed contraction in z + scatter-add ----------
  for (int w = tid; w < ne * N * N; w += NT) {
    const int i = w % N, j = (w / N) % N, el = w / (N * N);
    const int64_t e = e0 + el;
    const int ex = (int)(e % s.nx), ey = (int)((e / s.nx) % s.ny), ez = (int)(e / ((int64_t)s.nx * s.ny));
    const double* src = sZ + el * C::ZE + j * N + i;
    double X[3][NE], Y[3][NE];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int k = 0; k < NE; ++k) X[c][k] = Y[c][k] = 0.0;
#pragma unroll
    for (int a = 0; a < QE; ++a) {
      const bool mid = (Q & 1) && a == QH;
      double wbp[3], wbm[3], wdp[3], wdm[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double lb = src[c * C::ZC + a * C::SA], ld = src[c * C::ZC + C::ZV + a * C::SA];
        if (mid) {
          wbp[c] = lb; wdp[c] = ld; wbm[c] = wdm[c] = 0.0;
        } else {
          const double hb = src[c * C::ZC + (Q - 1 - a) * C::SA];
          const double hd = src[c * C::ZC + C::ZV + (Q - 1 - a) * C::SA];
          wbp[c] = lb + hb; wbm[c] = lb - hb;
          wdp[c] = ld + hd; wdm[c] = ld - hd;
        }
      }
#pragma unroll
      for (int k = 0; k < NE; ++k) {
        const bool kmid = (N & 1) && k == NH;
        const double be = tB[F::BE + k * QE + a];
        const double de = tD[F::BE + k * QE + a];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          X[c][k] = fma(be, wbp[c], X[c][k]);
          if (!kmid) Y[c][k] = fma(de, wdp[c], Y[c][k]);
        }
        if (!mid) {
          const double bo = tB[F::BO + k * QH + a];
          const double dO = tD[F::BO + k * QH + a];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            X[c][k] = fma(dO, wdm[c], X[c][k]);
            if (!kmid) Y[c][k] = fma(bo, wbm[c], Y[c][k]);
          }
        }
      }
    }
    const int I = ex * P + i, J = ey * P + j;
    const int64_t base = I + (int64_t)s.Nx * J + plane * ((int64_t)ez * P);
#pragma unroll
    for (int k = 0; k < NE; ++k) {
      const bool kmid = (N & 1) && k == NH;
      if (!(bc && is_constrained(I, J, ez * P + k, s))) {
#pragma unroll
        for (int c = 0; c < 3; ++c) atomicAdd(y + c * s.nodes + base + k * plane, kmid ? X[c][k] : X[c][k] + Y[c][k]);
      }
      if (!kmid && !(bc && is_constrained(I, J, ez * P + N - 1 - k, s))) {
#pragma unroll
        for (int c = 0; c < 3; ++c) atomicAdd(y + c * s.nodes + base + (N - 1 - k) * plane, X[c][k] - Y[c][k]);
      }
    }
  }
}

template <int P, int Q>
cudaError_t launch_apply_eo_pq(const Slab& s, const double* x, double* y, const double* qd, const double* rr,
                               const double* tables, int64_t e_begin, int64_t e_end, cudaStream_t st) {
  using C = CfgEO<P, Q>;
  static bool attr_done = false;
  static int pref = -1;
  if (!attr_done) {
    cudaError_t err = cudaFuncSetAttribute(apply_eo_kernel<P, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)C::smem);
    if (err != cudaSuccess) return err;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, apply_eo_kernel<P, Q>, C::NT, C::smem);
    pref = sms * (per_sm > 0 ? per_sm : 1);
    attr_done = true;
  }
  const int64_t ne = e_end - e_begin;
  if (ne <= 0) return cudaSuccess;
  const int64_t grid = (ne + C::EB - 1) / C::EB;
  apply_eo_kernel<P, Q><<<(unsigned)grid, C::NT, C::smem, st>>>(x, y, qd, rr, tables, s, e_begin, e_end, pref);
  return cudaGetLastError();
}

template <int P, int Q>
void info_eo_pq(ApplyLaunch* info) {
  using C = CfgEO<P, Q>;
  info->threads = C::NT;
  info->elems_per_cta = C::EB;
  info->smem_bytes = C::smem;
}

}  // namespace elas

#define ELAS_DEFINE_DEGREE_EO(P)                                                                \
  namespace elas {                                                                              \
  cudaError_t apply_eo_info_p##P(int q, ApplyLaunch* info) {                                    \
    if (q == P + 1) info_eo_pq<P, P + 1>(info);                                                 \
    else if (q == P + 2) info_eo_pq<P, P + 2>(info);                                            \
    else return cudaErrorInvalidValue;                                                          \
    return cudaSuccess;                                                                         \
  }                                                                                             \
  cudaError_t apply_eo_launch_p##P(int q, const Slab& s, const double* x, double* y,            \
                                   const double* qd, const double* rr, const double* tables,    \
                                   int64_t e_begin, int64_t e_end, cudaStream_t st) {           \
    if (q == P + 1) return launch_apply_eo_pq<P, P + 1>(s, x, y, qd, rr, tables, e_begin, e_end, st); \
    if (q == P + 2) return launch_apply_eo_pq<P, P + 2>(s, x, y, qd, rr, tables, e_begin, e_end, st); \
    return cudaErrorInvalidValue;                                                               \
  }                                                                                             \
  }
