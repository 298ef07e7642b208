// The paper's optimization stages on B200 (Sec. 5.4 "Ablation Study", Table 4):
// the same y = A x computed the way each stage of the ablation computes it, so the B200 cost of
// each step can be measured against the fused kernels (ELAS_VARIANT_ABL_*).
//
//   stage 0  "PA (baseline)", Alg. 1: element restriction E = G x (HBM), the
//            physical derivatives at every quadrature point from the dense basis-gradient matrix
//            Gm[pt][d][node] (O(p^6) per element, Gm streamed from memory), Kernel 1 writes the
//            transformed stress of every point to QVec (HBM, 9 values per point) with the full
//            3x3 strain/stress tensors, Kernel 2 contracts QVec with the dense Gm again
//            (Y_iqe += sum_pm QVec_pmqe G_pmi) and the element vectors are scattered into y.
//   stage 1  "+ Sum Factorization (C1)": both contractions as three
//            staged 1D contractions per element (one CTA per element, shared-memory staging);
//            QVec still round-trips through HBM.
//   stage 2  "+ Voigt Notation (C2)": Kernel 1 stores only the 6 unique
//            stress components per point (QVec 33 % smaller); Kernel 2 applies the geometric
//            transform F = sigma~ A~^T while loading them.
//   stages 3 and 4 ("+ Kernel Fusion (C3)", "+ Loop Structure") are the fused kernels:
//            ELAS_VARIANT_SIMT and ELAS_VARIANT_FOLDED (elas_apply.cuh, elas_apply_eo.cuh).
//
// Scaled form throughout: H = G A~ with A~ = sqrt(mu W) J^{-1} stored per
// point (QD_LAYOUT_LINES), sigma~ = r tr(eps) I + 2 eps with eps = (H + H^T)/2, r = lambda/mu, and
// F = sigma~ A~^T = W sigma J^{-T}.  All FP64.  Every kernel takes the element range [e0, e1).
#include "elas_internal.h"
#include "elas_apply.cuh"
#include "elas_op.h"

namespace elas {
namespace abl {

constexpr int NTE = 256;   // element-wise kernels
// threads of the one-CTA-per-element kernels: 512 where stage X has >= 512 fibres (9 q^2)
template <int N, int QQ> struct Ntc { static constexpr int value = 9 * QQ * QQ >= 512 ? 512 : 256; };
// elements per CTA: at p <= 5 enough stage-Y fibres (3 q n each) for the threads, within ~200 KB
// of shared memory (config 4: p2 23.1 -> 18.9 ms, p4 10.9 -> 9.7); one at p >= 6, where two would
// halve the resident threads
template <int N, int QQ, int PE>
struct Eba {
  static constexpr int want = N <= 6 ? Ntc<N, QQ>::value / (3 * QQ * N) : 1;
  static constexpr int cap = (200 * 1024 / 8) / PE;
  static constexpr int w1 = want < 1 ? 1 : (want > 8 ? 8 : want);
  static constexpr int value = w1 < cap ? w1 : (cap < 1 ? 1 : cap);
};
template <int N, int QQ> struct PeG {   // gradient kernel: Z1 | u / Y1 per element
  static constexpr int value = 6 * QQ * N * N + (3 * N * N * N > 9 * QQ * QQ * N ? 3 * N * N * N : 9 * QQ * QQ * N);
};
template <int N, int QQ> struct PeD {   // transposed kernel: F | T1 | T2 per element
  static constexpr int value = 9 * QQ * QQ * QQ + 9 * QQ * QQ * N + 6 * QQ * N * N;
};

__host__ __device__ inline int64_t grid_of(int64_t n, int nt) {
  const int64_t g = (n + nt - 1) / nt;
  return g < 1 ? 1 : (g > 1048576 ? 1048576 : g);
}

__device__ __forceinline__ int64_t node_index(const Slab& s, int64_t e, int i, int j, int k, int p, int& I, int& J,
                                              int& K) {
  const int ex = (int)(e % s.nx), ey = (int)((e / s.nx) % s.ny), ez = (int)(e / ((int64_t)s.nx * s.ny));
  I = ex * p + i;
  J = ey * p + j;
  K = ez * p + k;
  return I + (int64_t)s.Nx * (J + (int64_t)s.Ny * K);
}

// dense basis-gradient matrix Gm[(pt * 3 + d) * n^3 + node] = d/dxi_d phi_node at point pt (reference
// coordinates), from the 1D tables B (q x n) and D (q x n)
__global__ void gm_kernel(int n, int q, const double* __restrict__ tab, double* __restrict__ Gm) {
  const int n3 = n * n * n, q3 = q * q * q;
  const double* B = tab;
  const double* D = tab + q * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)q3 * 3 * n3;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int node = (int)(t % n3), d = (int)((t / n3) % 3), pt = (int)(t / (3 * n3));
    const int i = node % n, j = (node / n) % n, k = node / (n * n);
    const int a1 = pt % q, a2 = (pt / q) % q, a3 = pt / (q * q);
    const double fx = d == 0 ? D[a1 * n + i] : B[a1 * n + i];
    const double fy = d == 1 ? D[a2 * n + j] : B[a2 * n + j];
    const double fz = d == 2 ? D[a3 * n + k] : B[a3 * n + k];
    Gm[t] = fx * fy * fz;
  }
}

// E[e][c][node] = (Z x) restricted to element e
template <int N>
__global__ void gather_kernel(Slab s, const double* __restrict__ x, double* __restrict__ E, int64_t e0, int64_t e1) {
  constexpr int n = N, n3 = N * N * N, p = N - 1;
  const bool bc = s.faces != 0;
  for (int64_t t = e0 * 3 * n3 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < e1 * 3 * n3;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / (3 * n3);
    const int c = (int)((t / n3) % 3), node = (int)(t % n3);
    int I, J, K;
    const int64_t g = node_index(s, e, node % n, (node / n) % n, node / (n * n), p, I, J, K);
    E[t] = (bc && is_constrained(I, J, K, s)) ? 0.0 : x[c * s.nodes + g];
  }
}

// y[node] += Eo[e][c][node] on free rows (constrained rows hold (I - Z) x from the init)
template <int N>
__global__ void scatter_kernel(Slab s, const double* __restrict__ Eo, double* __restrict__ y, int64_t e0, int64_t e1) {
  constexpr int n = N, n3 = N * N * N, p = N - 1;
  const bool bc = s.faces != 0;
  for (int64_t t = e0 * 3 * n3 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < e1 * 3 * n3;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / (3 * n3);
    const int c = (int)((t / n3) % 3), node = (int)(t % n3);
    int I, J, K;
    const int64_t g = node_index(s, e, node % n, (node / n) % n, node / (n * n), p, I, J, K);
    if (!(bc && is_constrained(I, J, K, s))) atomicAdd(y + c * s.nodes + g, Eo[t]);
  }
}

// stage 0: reference gradients at every point from the dense Gm: Q[e][pt][3c + d]
template <int N, int QQ>
__global__ void grad_dense_kernel(const double* __restrict__ E, const double* __restrict__ Gm,
                                  double* __restrict__ Q, int64_t e0, int64_t e1) {
  constexpr int n3 = N * N * N, q3 = QQ * QQ * QQ;
  for (int64_t t = e0 * q3 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < e1 * q3;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / q3;
    const int pt = (int)(t % q3);
    const double* u = E + e * 3 * n3;
    const double* g = Gm + (int64_t)pt * 3 * n3;
    double G[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int node = 0; node < n3; ++node) {
      const double g0 = g[node], g1 = g[n3 + node], g2 = g[2 * n3 + node];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double uc = u[c * n3 + node];
        G[c][0] = fma(uc, g0, G[c][0]);
        G[c][1] = fma(uc, g1, G[c][1]);
        G[c][2] = fma(uc, g2, G[c][2]);
      }
    }
    double* o = Q + t * 9;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int d = 0; d < 3; ++d) o[3 * c + d] = G[c][d];
  }
}

// stage 0: Eo[e][c][node] = sum_pt sum_d F[e][pt][3c + d] Gm[pt][d][node]  (Alg. 1 Kernel 2)
template <int N, int QQ>
__global__ void div_dense_kernel(const double* __restrict__ Q, const double* __restrict__ Gm,
                                 double* __restrict__ Eo, int64_t e0, int64_t e1) {
  constexpr int n3 = N * N * N, q3 = QQ * QQ * QQ;
  for (int64_t t = e0 * 3 * n3 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < e1 * 3 * n3;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / (3 * n3);
    const int c = (int)((t / n3) % 3), node = (int)(t % n3);
    const double* F = Q + e * q3 * 9 + 3 * c;
    double acc = 0.0;
    for (int pt = 0; pt < q3; ++pt) {
      const double* g = Gm + (int64_t)pt * 3 * n3 + node;
      acc = fma(F[pt * 9 + 0], g[0], acc);
      acc = fma(F[pt * 9 + 1], g[n3], acc);
      acc = fma(F[pt * 9 + 2], g[2 * n3], acc);
    }
    Eo[t] = acc;
  }
}

// A~[d][m] of element e at point (a1, a2, a3), QD_LAYOUT_LINES
__device__ __forceinline__ void load_A(const double* __restrict__ qd, int q, int64_t e, int pt, double (&A)[9]) {
  const int a1 = pt % q, a2 = (pt / q) % q, a3 = pt / (q * q);
  const double* src = qd + e * (int64_t)qd_stride_lines(q) + (int64_t)a1 * 9 * q * q + (a3 + q * a2);
#pragma unroll
  for (int f = 0; f < 9; ++f) A[f] = src[f * q * q];
}

// Kernel 1 (pointwise).  voigt = 0: full 3x3 strain and stress tensors, stores F = sigma~ A~^T
// (9 per point, in place of the gradients); voigt = 1: the 6 unique stress components
// [s11, s22, s33, s23, s13, s12] (6 per point, packed at stride 9 so the gradient slot is reused)
template <int QQ>
__global__ void point_kernel(const double* __restrict__ qd, const double* __restrict__ rr,
                             double* __restrict__ Q, int voigt, int64_t e0, int64_t e1) {
  constexpr int q = QQ, q3 = QQ * QQ * QQ;
  for (int64_t t = e0 * q3 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < e1 * q3;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / q3;
    const int pt = (int)(t % q3);
    double A[9], G[3][3];
    load_A(qd, q, e, pt, A);
    double* o = Q + t * 9;
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int d = 0; d < 3; ++d) G[c][d] = o[3 * c + d];
    const double r = rr[e];
    double H[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int m = 0; m < 3; ++m) H[c][m] = fma(G[c][2], A[6 + m], fma(G[c][1], A[3 + m], G[c][0] * A[m]));
    if (voigt) {
      const double s = r * (H[0][0] + H[1][1] + H[2][2]);
      o[0] = fma(2.0, H[0][0], s);
      o[1] = fma(2.0, H[1][1], s);
      o[2] = fma(2.0, H[2][2], s);
      o[3] = H[1][2] + H[2][1];
      o[4] = H[0][2] + H[2][0];
      o[5] = H[0][1] + H[1][0];
    } else {
      double eps[3][3], sig[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) eps[i][j] = 0.5 * (H[i][j] + H[j][i]);
      const double tr = eps[0][0] + eps[1][1] + eps[2][2];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) sig[i][j] = (i == j ? r * tr : 0.0) + 2.0 * eps[i][j];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d)
          o[3 * c + d] = fma(sig[c][2], A[3 * d + 2], fma(sig[c][1], A[3 * d + 1], sig[c][0] * A[3 * d]));
    }
  }
}

// stages 1-2: forward sum factorisation, one CTA per element:
//   Z1[c][zk][a3][j][i] = sum_k (zk ? D : B)[a3][k] u[c][k][j][i]
//   Y1[c][d][a3][a2][i] = sum_j (d == 1 ? D : B)[a2][j] Z1[c][d == 2][a3][j][i]
//   G[c][d](a1, a2, a3) = sum_i (d == 0 ? D : B)[a1][i] Y1[c][d][a3][a2][i]   -> Q[e][pt][3c + d]
template <int N, int QQ>
__global__ void __launch_bounds__(Ntc<N, QQ>::value, 1) grad_sf_kernel(const double* __restrict__ E, const double* __restrict__ tab,
                                                      double* __restrict__ Q, int64_t e0, int64_t e1) {
  extern __shared__ double sm[];
  constexpr int n = N, q = QQ, n2 = n * n, n3 = n2 * n, q2 = q * q, q3 = q2 * q, NTC = Ntc<N, QQ>::value;
  constexpr int PE = PeG<N, QQ>::value, EB = Eba<N, QQ, PE>::value;
  double* B = sm;
  double* D = B + q * n;
  // per element el: Z1 = D + q n + el PE (3 * 2 * q * n^2), then u (3 n^3, dead after stage Z, so
  // stage Y writes Y1 = 3 * 3 * q^2 * n over it)
#define ABL_Z1(el) (D + q * n + (el) * PE)
#define ABL_U(el) (ABL_Z1(el) + 6 * q * n2)
  const int64_t eb = e0 + (int64_t)blockIdx.x * EB;
  const int ne = (int)((e1 - eb) < EB ? (e1 - eb) : EB);
  for (int t = threadIdx.x; t < 2 * q * n; t += NTC) sm[t] = tab[t];
  for (int t = threadIdx.x; t < ne * 3 * n3; t += NTC) ABL_U(t / (3 * n3))[t % (3 * n3)] = E[eb * 3 * n3 + t];
  __syncthreads();
  // one thread per 1D fibre, its n (or q) inputs loaded once into registers
  for (int t = threadIdx.x; t < ne * 3 * n2; t += NTC) {            // stage Z: fibre (c, j, i)
    const int el = t / (3 * n2), ji = t % n2, c = (t / n2) % 3;
    const double* u = ABL_U(el);
    double* Z1 = ABL_Z1(el);
    double v[n];
#pragma unroll
    for (int k = 0; k < n; ++k) v[k] = u[c * n3 + k * n2 + ji];
#pragma unroll 1   // coefficients reloaded per output (hoisting them all spills)
    for (int a3 = 0; a3 < q; ++a3) {
      double sb = 0.0, sd = 0.0;
#pragma unroll
      for (int k = 0; k < n; ++k) {
        sb = fma(B[a3 * n + k], v[k], sb);
        sd = fma(D[a3 * n + k], v[k], sd);
      }
      Z1[((c * 2 + 0) * q + a3) * n2 + ji] = sb;
      Z1[((c * 2 + 1) * q + a3) * n2 + ji] = sd;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < ne * 3 * q * n; t += NTC) {         // stage Y: fibre (c, a3, i)
    const int el = t / (3 * q * n), i = t % n, a3 = (t / n) % q, c = (t / (n * q)) % 3;
    const double* Z1 = ABL_Z1(el);
    double* Y1 = ABL_U(el);
    double vb[n], vd[n];
#pragma unroll
    for (int j = 0; j < n; ++j) {
      vb[j] = Z1[((c * 2 + 0) * q + a3) * n2 + j * n + i];
      vd[j] = Z1[((c * 2 + 1) * q + a3) * n2 + j * n + i];
    }
#pragma unroll 1   // coefficients reloaded per output (hoisting them all spills)
    for (int a2 = 0; a2 < q; ++a2) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int j = 0; j < n; ++j) {
        s0 = fma(B[a2 * n + j], vb[j], s0);
        s1 = fma(D[a2 * n + j], vb[j], s1);
        s2 = fma(B[a2 * n + j], vd[j], s2);
      }
      Y1[(((c * 3 + 0) * q + a3) * q + a2) * n + i] = s0;
      Y1[(((c * 3 + 1) * q + a3) * q + a2) * n + i] = s1;
      Y1[(((c * 3 + 2) * q + a3) * q + a2) * n + i] = s2;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < ne * 9 * q2; t += NTC) {            // stage X: fibre (c, d, a3, a2)
    const int el = t / (9 * q2), a2 = t % q, a3 = (t / q) % q, cd = (t / q2) % 9;
    const int64_t e = eb + el;
    const double* Y1 = ABL_U(el);
    const double* T = (cd % 3) == 0 ? D : B;
    double v[n];
#pragma unroll
    for (int i = 0; i < n; ++i) v[i] = Y1[((cd * q + a3) * q + a2) * n + i];
#pragma unroll 1   // coefficients reloaded per output (hoisting them all spills)
    for (int a1 = 0; a1 < q; ++a1) {
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < n; ++i) acc = fma(T[a1 * n + i], v[i], acc);
      Q[(e * q3 + a1 + q * (a2 + q * a3)) * 9 + cd] = acc;
    }
  }
}

#undef ABL_Z1
#undef ABL_U

// stages 1-2: transposed sum factorisation (Alg. 1 Kernel 2 with C1), one CTA per element.
// voigt = 1: Q holds the 6 stress components; F = sigma~ A~^T is formed on load from qdata.
//   T1[c][d][a3][a2][i] = sum_a1 (d == 0 ? D : B)[a1][i] F[c][d](a1, a2, a3)
//   T2[c][zk][a3][j][i] = zk = 0: sum_a2 B[a2][j] T1[c][0] + D[a2][j] T1[c][1];  zk = 1: sum_a2 B[a2][j] T1[c][2]
//   Eo[c][k][j][i]      = sum_a3 B[a3][k] T2[c][0] + D[a3][k] T2[c][1]
template <int N, int QQ>
__global__ void __launch_bounds__(Ntc<N, QQ>::value, 1) div_sf_kernel(const double* __restrict__ Q, const double* __restrict__ qd,
                                                     const double* __restrict__ tab, double* __restrict__ Eo, int voigt,
                                                     int64_t e0, int64_t e1) {
  extern __shared__ double sm[];
  constexpr int n = N, q = QQ, n2 = n * n, n3 = n2 * n, q2 = q * q, q3 = q2 * q, NTC = Ntc<N, QQ>::value;
  constexpr int PE = PeD<N, QQ>::value, EB = Eba<N, QQ, PE>::value;
  double* B = sm;
  double* D = B + q * n;
  // per element el: F ([c][d][pt], 9 q^3) | T1 (9 q^2 n) | T2 (6 q n^2)
#define ABL_F(el) (D + q * n + (el) * PE)
#define ABL_T1(el) (ABL_F(el) + 9 * q3)
#define ABL_T2(el) (ABL_T1(el) + 9 * q2 * n)
  const int64_t eb = e0 + (int64_t)blockIdx.x * EB;
  const int ne = (int)((e1 - eb) < EB ? (e1 - eb) : EB);
  for (int t = threadIdx.x; t < 2 * q * n; t += NTC) sm[t] = tab[t];
  if (voigt) {
    for (int t = threadIdx.x; t < ne * q3; t += NTC) {
      const int el = t / q3, pt = t % q3;
      const int64_t e = eb + el;
      double* F = ABL_F(el);
      const double* sv = Q + (e * q3 + pt) * 9;
      const double S[3][3] = {{sv[0], sv[5], sv[4]}, {sv[5], sv[1], sv[3]}, {sv[4], sv[3], sv[2]}};
      double A[9];
      load_A(qd, q, e, pt, A);
      for (int c = 0; c < 3; ++c)
        for (int d = 0; d < 3; ++d)
          F[(c * 3 + d) * q3 + pt] = fma(S[c][2], A[3 * d + 2], fma(S[c][1], A[3 * d + 1], S[c][0] * A[3 * d]));
    }
  } else {
    for (int t = threadIdx.x; t < ne * 9 * q3; t += NTC) {
      const int el = t / (9 * q3), cd = t % 9, pt = (t / 9) % q3;
      ABL_F(el)[cd * q3 + pt] = Q[eb * q3 * 9 + t];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < ne * 9 * q2; t += NTC) {            // stage Xt: fibre (c, d, a3, a2)
    const int el = t / (9 * q2), a2 = t % q, a3 = (t / q) % q, cd = (t / q2) % 9;
    const double* F = ABL_F(el);
    double* T1 = ABL_T1(el);
    const double* T = (cd % 3) == 0 ? D : B;
    double v[q];
#pragma unroll
    for (int a1 = 0; a1 < q; ++a1) v[a1] = F[cd * q3 + (a3 * q + a2) * q + a1];
#pragma unroll 1   // coefficients reloaded per output (hoisting them all spills)
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int a1 = 0; a1 < q; ++a1) acc = fma(T[a1 * n + i], v[a1], acc);
      T1[((cd * q + a3) * q + a2) * n + i] = acc;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < ne * 3 * q * n; t += NTC) {         // stage Yt: fibre (c, a3, i)
    const int el = t / (3 * q * n), i = t % n, a3 = (t / n) % q, c = (t / (n * q)) % 3;
    const double* T1 = ABL_T1(el);
    double* T2 = ABL_T2(el);
    double v0[q], v1[q], v2[q];
#pragma unroll
    for (int a2 = 0; a2 < q; ++a2) {
      v0[a2] = T1[(((c * 3 + 0) * q + a3) * q + a2) * n + i];
      v1[a2] = T1[(((c * 3 + 1) * q + a3) * q + a2) * n + i];
      v2[a2] = T1[(((c * 3 + 2) * q + a3) * q + a2) * n + i];
    }
#pragma unroll 1   // coefficients reloaded per output (hoisting them all spills)
    for (int j = 0; j < n; ++j) {
      double sb = 0.0, sd = 0.0;
#pragma unroll
      for (int a2 = 0; a2 < q; ++a2) {
        sb = fma(B[a2 * n + j], v0[a2], fma(D[a2 * n + j], v1[a2], sb));
        sd = fma(B[a2 * n + j], v2[a2], sd);
      }
      T2[((c * 2 + 0) * q + a3) * n2 + j * n + i] = sb;
      T2[((c * 2 + 1) * q + a3) * n2 + j * n + i] = sd;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < ne * 3 * n2; t += NTC) {            // stage Zt: fibre (c, j, i)
    const int el = t / (3 * n2), ji = t % n2, c = (t / n2) % 3;
    const int64_t e = eb + el;
    const double* T2 = ABL_T2(el);
    double vb[q], vd[q];
#pragma unroll
    for (int a3 = 0; a3 < q; ++a3) {
      vb[a3] = T2[((c * 2 + 0) * q + a3) * n2 + ji];
      vd[a3] = T2[((c * 2 + 1) * q + a3) * n2 + ji];
    }
#pragma unroll 1   // coefficients reloaded per output (hoisting them all spills)
    for (int k = 0; k < n; ++k) {
      double acc = 0.0;
#pragma unroll
      for (int a3 = 0; a3 < q; ++a3) acc = fma(B[a3 * n + k], vb[a3], fma(D[a3 * n + k], vd[a3], acc));
      Eo[e * 3 * n3 + c * n3 + k * n2 + ji] = acc;
    }
  }
}

#undef ABL_F
#undef ABL_T1
#undef ABL_T2

template <int N, int QQ>
size_t grad_sf_smem() { return sizeof(double) * (2 * QQ * N + (size_t)Eba<N, QQ, PeG<N, QQ>::value>::value * PeG<N, QQ>::value); }
template <int N, int QQ>
size_t div_sf_smem() { return sizeof(double) * (2 * QQ * N + (size_t)Eba<N, QQ, PeD<N, QQ>::value>::value * PeD<N, QQ>::value); }

template <int N, int QQ>
cudaError_t run_stage(const elas_op* op, int stage, const double* x, double* y, int64_t e0, int64_t e1, cudaStream_t st,
                      bool first) {
  constexpr int n3 = N * N * N, q3 = QQ * QQ * QQ;
  cudaError_t err;
  (void)first;
  // per-device function attributes: set on the current device on every call (not a hot path)
  if ((err = cudaFuncSetAttribute(grad_sf_kernel<N, QQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)) ||
      (err = cudaFuncSetAttribute(div_sf_kernel<N, QQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)))
    return err;
  const Slab& s = op->slab;
  const int64_t nel = e1 - e0;
  gather_kernel<N><<<(unsigned)grid_of(nel * 3 * n3, NTE), NTE, 0, st>>>(s, x, op->abl_E, e0, e1);
  if (stage == 0)
    grad_dense_kernel<N, QQ><<<(unsigned)grid_of(nel * q3, NTE), NTE, 0, st>>>(op->abl_E, op->abl_G, op->abl_Q, e0, e1);
  else {
    constexpr int EB = Eba<N, QQ, PeG<N, QQ>::value>::value;
    grad_sf_kernel<N, QQ><<<(unsigned)((nel + EB - 1) / EB), Ntc<N, QQ>::value, grad_sf_smem<N, QQ>(), st>>>(
        op->abl_E, op->tab, op->abl_Q, e0, e1);
  }
  point_kernel<QQ><<<(unsigned)grid_of(nel * q3, NTE), NTE, 0, st>>>(op->qd, op->rr, op->abl_Q, stage >= 2, e0, e1);
  if (stage == 0)
    div_dense_kernel<N, QQ><<<(unsigned)grid_of(nel * 3 * n3, NTE), NTE, 0, st>>>(op->abl_Q, op->abl_G, op->abl_Eo, e0, e1);
  else {
    constexpr int EB = Eba<N, QQ, PeD<N, QQ>::value>::value;
    div_sf_kernel<N, QQ><<<(unsigned)((nel + EB - 1) / EB), Ntc<N, QQ>::value, div_sf_smem<N, QQ>(), st>>>(
        op->abl_Q, op->qd, op->tab, op->abl_Eo, stage >= 2, e0, e1);
  }
  scatter_kernel<N><<<(unsigned)grid_of(nel * 3 * n3, NTE), NTE, 0, st>>>(s, op->abl_Eo, y, e0, e1);
  return cudaGetLastError();
}

template <int P>
cudaError_t run_p(const elas_op* op, int stage, const double* x, double* y, int64_t e0, int64_t e1, cudaStream_t st,
                  bool first) {
  if (op->q == P + 1) return run_stage<P + 1, P + 1>(op, stage, x, y, e0, e1, st, first);
  if (op->q == P + 2) return run_stage<P + 1, P + 2>(op, stage, x, y, e0, e1, st, first);
  return cudaErrorInvalidValue;
}

}  // namespace abl

// One pass of ablation stage `stage` (0, 1, 2) over the elements [e0, e1): gather -> gradients ->
// pointwise -> transposed contraction -> scatter (5 launches).  Scratch (E-vectors, QVec, Gm) is
// allocated on first use and owned by the op.
cudaError_t ablation_apply(elas_op* op, int stage, const double* x, double* y, int64_t e0, int64_t e1, cudaStream_t st) {
  using namespace abl;
  if (e1 <= e0) return cudaSuccess;
  const Slab& s = op->slab;
  const int p = op->p, q = op->q, n = p + 1, n3 = n * n * n, q3 = q * q * q;
  const int64_t ne = (int64_t)s.nx * s.ny * s.nz;
  cudaError_t err;
  const bool first = !(op->abl_E && op->abl_Eo && op->abl_Q && op->abl_G);
  if (first) {
    if ((err = cudaMalloc(&op->abl_E, sizeof(double) * 3 * n3 * ne)) ||
        (err = cudaMalloc(&op->abl_Eo, sizeof(double) * 3 * n3 * ne)) ||
        (err = cudaMalloc(&op->abl_Q, sizeof(double) * 9 * (size_t)q3 * ne)) ||
        (err = cudaMalloc(&op->abl_G, sizeof(double) * (size_t)q3 * 3 * n3))) {
      // all or nothing: a later call must not find part of the scratch and skip the allocation
      for (double** b : {&op->abl_E, &op->abl_Eo, &op->abl_Q, &op->abl_G}) {
        if (*b) cudaFree(*b);
        *b = nullptr;
      }
      return err;
    }
    gm_kernel<<<(unsigned)grid_of((int64_t)q3 * 3 * n3, NTE), NTE, 0, st>>>(n, q, op->tab, op->abl_G);
    if ((err = cudaGetLastError())) return err;
  }
  switch (p) {
    case 1: return run_p<1>(op, stage, x, y, e0, e1, st, first);
    case 2: return run_p<2>(op, stage, x, y, e0, e1, st, first);
    case 3: return run_p<3>(op, stage, x, y, e0, e1, st, first);
    case 4: return run_p<4>(op, stage, x, y, e0, e1, st, first);
    case 5: return run_p<5>(op, stage, x, y, e0, e1, st, first);
    case 6: return run_p<6>(op, stage, x, y, e0, e1, st, first);
    case 7: return run_p<7>(op, stage, x, y, e0, e1, st, first);
    case 8: return run_p<8>(op, stage, x, y, e0, e1, st, first);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace elas
