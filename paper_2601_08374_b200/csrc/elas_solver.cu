// Consumers of the apply in the paper's solver (PAPER.md:202-210,
// Sec. 3.1; SPEC.md solvers): the matrix-free operator diagonal, the power-iteration estimate
// of lambda_max(D^{-1} A), the Chebyshev polynomial smoother and preconditioned CG.  Every step
// runs in the kernels below or in elas_apply; the host only sequences launches and reads the
// scalar it needs for the convergence test.
//
// * diag_kernel (setup-time, one CTA per element): with h = grad_xi phi_I . A~ (A~ = sqrt(mu W)
//   J^{-1}, the stored qdata), A[(c,I),(c,I)] = sum_qp (1 + r) h_c^2 + |h|^2 (r = lambda/mu).
//   Expanding h_c^2 = sum_kl g_k g_l A~_kc A~_lc (g_k = d phi_I / d xi_k = a product of 1D B/D
//   factors) gives, for each of the 6 pairs k <= l, a q^3 tensor
//   M_c,kl = (1 + r) A~_kc A~_lc + (A~ A~^T)_kl contracted with the 1D product tables
//   F_d,kl[a][i] = T_k^d[a][i] T_l^d[a][i] (T_k^d = D if k == d else B) along x, y, z in turn
//   (sum factorisation of the diagonal, O(q^3 n) per tensor).
// * Chebyshev (Saad, Iterative Methods, Alg. 12.1) on D^{-1} A for [alpha lam, beta lam]:
//   two fused vector kernels per step around elas_apply.
// * PCG: dots by a deterministic two-pass reduction into device scalars; alpha and beta are
//   formed on the device inside the update kernels (no host round trip but the convergence
//   read of r.z, 8 bytes per iteration).
#include <cmath>
#include <cstdio>
#include <string>

#include "elas_op.h"

namespace elas {
namespace {

constexpr int RED_BLOCKS = 296;    // 2 x 148 SMs; fixed so the reduction order is fixed
constexpr int RED_THREADS = 256;
// device scalar slots after the RED_BLOCKS partials
enum { S_DOT = 0, S_RZ, S_RZNEW, S_PT, S_NRM, S_LAM, S_ZT, S_COUNT };

int fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? ELAS_ENOMEM : ELAS_ECUDA;
}
#define CK(expr, what)                                \
  do {                                                \
    cudaError_t e_ = (expr);                          \
    if (e_ != cudaSuccess) return fail(e_, what);     \
  } while (0)

#define CK_C(expr, what)                                      \
  do {                                                        \
    cudaError_t e_ = (expr);                                  \
    if (e_ != cudaSuccess) return elas::fail(e_, what);       \
  } while (0)

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

__device__ __forceinline__ bool cons_node(int64_t node, const Slab& s) {
  const int I = (int)(node % s.Nx), J = (int)((node / s.Nx) % s.Ny), K = (int)(node / ((int64_t)s.Nx * s.Ny));
  const uint32_t f = s.faces;
  return ((f & ELAS_FACE_XMIN) && I == 0) || ((f & ELAS_FACE_XMAX) && I == s.Nx - 1) ||
         ((f & ELAS_FACE_YMIN) && J == 0) || ((f & ELAS_FACE_YMAX) && J == s.Ny - 1) ||
         ((f & ELAS_FACE_ZMIN) && K == 0) || ((f & ELAS_FACE_ZMAX) && K == s.Nz - 1);
}

// ------------------------------------------------------------------------- diagonal

// word offset of A~[0] (f = 3 k + m at + f * fstride) at point (a1, a2, a3) of element e, for
// every qdata layout (QD_LAYOUT_LINES_F32 holds floats; the caller reads accordingly)
__device__ __forceinline__ int64_t qd_offset(int layout, int q, int64_t e, int a1, int a2, int a3, int& fstride) {
  const int q3 = q * q * q;
  if (layout == QD_LAYOUT_E32) {
    fstride = 32;
    const int pt = a1 + q * (a2 + q * a3);
    return (e >> 5) * (int64_t)(32 * 9 * q3) + (int64_t)pt * 9 * 32 + (e & 31);
  }
  if (layout == QD_LAYOUT_TC6) {
    fstride = 32;
    const int sl = a1 >> 1, r = 2 * (a1 & 1) + (a3 & 1), lane = 4 * a2 + (a3 >> 1);
    return e * (int64_t)(9 * q3) + (int64_t)((sl * 4 + r) * 9) * 32 + lane;
  }
  fstride = q * q;
  const int64_t es = layout == QD_LAYOUT_LINES_F32 ? (int64_t)((9 * q3 + 3) & ~3) : (int64_t)qd_stride_lines(q);
  return e * es + (int64_t)a1 * 9 * q * q + a3 + q * a2;
}

// A~ at point (a1, a2, a3) from the geometry-on-the-fly coefficients (QD_LAYOUT_OTF)
__device__ __forceinline__ void otf_A(const double* ge, int st, const double* g, const double* sw, int a1, int a2,
                                      int a3, double (&A)[9]) {
  const double x1 = g[a1], x2 = g[a2], x3 = g[a3];
  double J[3][3];
  for (int m = 0; m < 3; ++m) {
    J[m][0] = ge[m * st] + ge[(3 + m) * st] * x2 + ge[(6 + m) * st] * x3 + ge[(9 + m) * st] * x2 * x3;
    J[m][1] = ge[(12 + m) * st] + ge[(15 + m) * st] * x1 + ge[(18 + m) * st] * x3 + ge[(21 + m) * st] * x1 * x3;
    J[m][2] = ge[(24 + m) * st] + ge[(27 + m) * st] * x1 + ge[(30 + m) * st] * x2 + ge[(33 + m) * st] * x1 * x2;
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
  const double sc = ge[36 * st] * sw[a1] * sw[a2] * sw[a3] * rsqrt(det);
  for (int d = 0; d < 3; ++d)
    for (int m = 0; m < 3; ++m) A[3 * d + m] = sc * adj[d][m];
}

__global__ void diag_init_kernel(Slab s, double* __restrict__ d) {
  const int64_t n = 3 * s.nodes;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    d[t] = (s.faces && cons_node(t % s.nodes, s)) ? 1.0 : 0.0;
}

// dynamic smem: B, D (q n each), F[3] (q n each), T0[3][q^3], T1[3][q^2 n], T2[3][q n^2], acc[3][n^3]
__global__ void __launch_bounds__(128) diag_kernel(int p, int q, int layout, Slab s, const double* __restrict__ qd,
                                                   const double* __restrict__ rr, const double* __restrict__ tables,
                                                   const double* __restrict__ gauss, const double* __restrict__ cc,
                                                   double* __restrict__ d) {
  extern __shared__ double sm[];
  const int n = p + 1, qn = q * n, q3 = q * q * q, n3 = n * n * n;
  double* sB = sm;
  double* sD = sB + qn;
  double* F = sD + qn;              // F[dir][a][i]
  double* T0 = F + 3 * qn;          // [c][a3][a2][a1]
  double* T1 = T0 + 3 * q3;         // [c][a3][a2][i]
  double* T2 = T1 + 3 * q * q * n;  // [c][a3][j][i]
  double* acc = T2 + 3 * q * n * n; // [c][k][j][i]
  const int tid = threadIdx.x, NT = blockDim.x;
  const int64_t e = blockIdx.x;
  for (int t = tid; t < 2 * qn; t += NT) sm[t] = tables[t];
  for (int t = tid; t < 3 * n3; t += NT) acc[t] = 0.0;
  const double r1 = 1.0 + rr[e];
  for (int kl = 0; kl < 6; ++kl) {
    const int k = kl < 3 ? kl : (kl == 3 ? 0 : (kl == 4 ? 0 : 1));
    const int l = kl < 3 ? kl : (kl == 3 ? 1 : 2);
    const double mult = (k == l) ? 1.0 : 2.0;
    __syncthreads();   // tables loaded / previous pass done with F, T*
    for (int t = tid; t < 3 * qn; t += NT) {
      const int dir = t / qn, ai = t % qn;
      const double fk = (k == dir) ? sD[ai] : sB[ai];
      const double fl = (l == dir) ? sD[ai] : sB[ai];
      F[t] = fk * fl;
    }
    for (int pt = tid; pt < q3; pt += NT) {
      const int a1 = pt % q, a2 = (pt / q) % q, a3 = pt / (q * q);
      double Ak[3], Al[3];
      if (layout == QD_LAYOUT_OTF || layout == QD_LAYOUT_OTF32) {
        double A[9];
        if (layout == QD_LAYOUT_OTF) otf_A(qd + e * (int64_t)GEO_WORDS, 1, gauss, gauss + q, a1, a2, a3, A);
        else otf_A(qd + (e >> 5) * (int64_t)(32 * GEO_WORDS) + (e & 31), 32, gauss, gauss + q, a1, a2, a3, A);
        for (int m = 0; m < 3; ++m) {
          Ak[m] = A[3 * k + m];
          Al[m] = A[3 * l + m];
        }
      } else {
        int fs;
        const int64_t off = qd_offset(layout, q, e, a1, a2, a3, fs);
        const float* qf = reinterpret_cast<const float*>(qd);
        const bool f32 = layout == QD_LAYOUT_LINES_F32;
        for (int m = 0; m < 3; ++m) {
          const int64_t ik = off + (3 * k + m) * fs, il = off + (3 * l + m) * fs;
          Ak[m] = f32 ? (double)qf[ik] : qd[ik];
          Al[m] = f32 ? (double)qf[il] : qd[il];
        }
      }
      if (cc) {   // anisotropic (Eq. 2): M_c,kl = sum_mn A~_km A~_ln C_cmcn, C from 21 Voigt words
        const double* C = cc + e * 21;
        const int V[3][3] = {{0, 5, 4}, {5, 1, 3}, {4, 3, 2}};
        for (int c = 0; c < 3; ++c) {
          double v = 0.0;
          for (int m = 0; m < 3; ++m)
            for (int n2 = 0; n2 < 3; ++n2) {
              const int a = V[c][m], b = V[c][n2];
              const int ia = a <= b ? a * 6 - a * (a - 1) / 2 + (b - a) : b * 6 - b * (b - 1) / 2 + (a - b);
              v = fma(Ak[m] * Al[n2], C[ia], v);
            }
          T0[c * q3 + pt] = v;
        }
      } else {
        const double dot = Ak[0] * Al[0] + Ak[1] * Al[1] + Ak[2] * Al[2];
        for (int c = 0; c < 3; ++c) T0[c * q3 + pt] = r1 * Ak[c] * Al[c] + dot;
      }
    }
    __syncthreads();
    for (int t = tid; t < 3 * q * q * n; t += NT) {   // x: a1 -> i
      const int i = t % n, a2 = (t / n) % q, a3 = (t / (n * q)) % q, c = t / (n * q * q);
      const double* src = T0 + c * q3 + (a3 * q + a2) * q;
      double v = 0.0;
      for (int a1 = 0; a1 < q; ++a1) v = fma(F[a1 * n + i], src[a1], v);
      T1[t] = v;
    }
    __syncthreads();
    for (int t = tid; t < 3 * q * n * n; t += NT) {   // y: a2 -> j
      const int i = t % n, j = (t / n) % n, a3 = (t / (n * n)) % q, c = t / (n * n * q);
      const double* src = T1 + ((c * q + a3) * q) * n + i;
      double v = 0.0;
      for (int a2 = 0; a2 < q; ++a2) v = fma(F[qn + a2 * n + j], src[a2 * n], v);
      T2[t] = v;
    }
    __syncthreads();
    for (int t = tid; t < 3 * n3; t += NT) {          // z: a3 -> k
      const int i = t % n, j = (t / n) % n, kk = (t / (n * n)) % n, c = t / n3;
      const double* src = T2 + (c * q) * n * n + j * n + i;
      double v = 0.0;
      for (int a3 = 0; a3 < q; ++a3) v = fma(F[2 * qn + a3 * n + kk], src[a3 * n * n], v);
      acc[t] = fma(mult, v, acc[t]);
    }
  }
  __syncthreads();
  const int ex = (int)(e % s.nx), ey = (int)((e / s.nx) % s.ny), ez = (int)(e / ((int64_t)s.nx * s.ny));
  for (int t = tid; t < 3 * n3; t += NT) {
    const int i = t % n, j = (t / n) % n, kk = (t / (n * n)) % n, c = t / n3;
    const int64_t node = (ex * p + i) + (int64_t)s.Nx * ((ey * p + j) + (int64_t)s.Ny * (ez * p + kk));
    if (s.faces && cons_node(node, s)) continue;
    atomicAdd(d + c * s.nodes + node, acc[t]);
  }
}

// ------------------------------------------------------------------------- reductions

// partial[b] = sum over this block's grid-stride share of w_i a_i b_i (w_i = 0 on interface
// planes owned by the rank below; none for one rank)
// One-launch deterministic dot: every block writes its partial of sum_c sum_{node >= skip} a b
// (skip = one node plane on ranks > 0 of a slab partition: the lower interface plane is
// replicated and owned by the rank below), and the LAST block to finish (atomic ticket) sums the
// RED_BLOCKS partials in a fixed tree order into *out and re-arms the ticket.
__global__ void __launch_bounds__(RED_THREADS) dot_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                          int64_t nodes, int64_t skip, double* __restrict__ partial,
                                                          double* __restrict__ out, unsigned int* __restrict__ ticket) {
  __shared__ double sh[RED_THREADS];
  __shared__ bool last;
  double v = 0.0;
  for (int c = 0; c < 3; ++c) {
    const double* ac = a + c * nodes;
    const double* bc = b + c * nodes;
    for (int64_t t = skip + blockIdx.x * (int64_t)RED_THREADS + threadIdx.x; t < nodes;
         t += (int64_t)RED_BLOCKS * RED_THREADS)
      v = fma(ac[t], bc[t], v);
  }
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int w = RED_THREADS / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = sh[0];
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double w = 0.0;
  for (int bb = threadIdx.x; bb < RED_BLOCKS; bb += RED_THREADS) w += ((volatile double*)partial)[bb];
  sh[threadIdx.x] = w;
  __syncthreads();
  for (int k = RED_THREADS / 2; k > 0; k >>= 1) {
    if ((int)threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *out = sh[0];
    *ticket = 0u;
  }
}

// distributed dot over the owned dofs of this rank, result in the device scalar `slot`
// (allreduced over the slab communicator in NCCL mode)
int dot(elas_op* op, const double* a, const double* b, int slot) {
  const Slab& s = op->slab;
  cudaStream_t st = op->stream;
  const int64_t skip = op->rank > 0 ? (int64_t)s.Nx * s.Ny : 0;
  dot_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(a, b, s.nodes, skip, op->red, op->red + RED_BLOCKS + slot,
                                                reinterpret_cast<unsigned int*>(op->red + RED_BLOCKS + S_COUNT));
  CK(cudaGetLastError(), "dot kernels");
  if (op->comm) {
    ncclResult_t r = ncclAllReduce(op->red + RED_BLOCKS + slot, op->red + RED_BLOCKS + slot, 1, ncclDouble, ncclSum,
                                   op->comm, st);
    if (r != ncclSuccess) {
      set_error(std::string("ncclAllReduce (dot): ") + ncclGetErrorString(r));
      return ELAS_ENCCL;
    }
  }
  return ELAS_OK;
}

// ------------------------------------------------------------------------- vector kernels

__global__ void inv_kernel(const double* __restrict__ d, double* __restrict__ dinv, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    dinv[t] = 1.0 / d[t];
}

// v <- s v / sqrt(S[nrm]),  s = 1
__global__ void normalize_kernel(double* __restrict__ v, const double* __restrict__ src, const double* __restrict__ S,
                                 int64_t n) {
  const double sc = 1.0 / sqrt(S[0]);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    v[t] = src[t] * sc;
}

// w = dinv * t
__global__ void scale_kernel(double* __restrict__ w, const double* __restrict__ dinv, const double* __restrict__ t_,
                             int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    w[t] = dinv[t] * t_[t];
}

// Chebyshev start: r = dinv (b - Ax) (Ax == nullptr: x = 0), dv = r / theta, x += dv (or x = dv)
__global__ void cheb_start_kernel(const double* __restrict__ b, const double* __restrict__ Ax,
                                  const double* __restrict__ dinv, double* __restrict__ r, double* __restrict__ dv,
                                  double* __restrict__ x, double inv_theta, int zero_x, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const double rt = dinv[t] * (Ax ? b[t] - Ax[t] : b[t]);
    const double d = rt * inv_theta;
    r[t] = rt;
    dv[t] = d;
    x[t] = zero_x ? d : x[t] + d;
  }
}

// Chebyshev step: r -= dinv Ad; dv = c1 dv + c2 r; x += dv
__global__ void cheb_step_kernel(const double* __restrict__ Ad, const double* __restrict__ dinv,
                                 double* __restrict__ r, double* __restrict__ dv, double* __restrict__ x, double c1,
                                 double c2, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const double rt = r[t] - dinv[t] * Ad[t];
    const double d = fma(c1, dv[t], c2 * rt);
    r[t] = rt;
    dv[t] = d;
    x[t] += d;
  }
}

// PCG: alpha = S[RZ] / S[PT]; x += alpha p; r -= alpha t; (jacobi) z = dinv r
__global__ void pcg_update_kernel(double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
                                  const double* __restrict__ p, const double* __restrict__ t_,
                                  const double* __restrict__ dinv, const double* __restrict__ S, int64_t n) {
  const double alpha = S[S_PT] != 0.0 ? S[S_RZ] / S[S_PT] : 0.0;   // 0/0 only for b = 0 or exact convergence
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    x[t] = fma(alpha, p[t], x[t]);
    const double rt = fma(-alpha, t_[t], r[t]);
    r[t] = rt;
    if (z) z[t] = dinv ? dinv[t] * rt : rt;
  }
}

// PCG: beta = S[RZNEW] / S[RZ] (Fletcher-Reeves), or with a variable preconditioner (flexible CG,
// Polak-Ribiere form) beta = z_new.(r_new - r_old) / rz_old = -(z_new.t) / (p.t), using
// r_old = r_new + alpha t and alpha = rz_old / (p.t); p = z + beta p; then S[RZ] = S[RZNEW]
__global__ void pcg_direction_kernel(double* __restrict__ p, const double* __restrict__ z, double* __restrict__ S,
                                     int64_t n, int first, int flexible) {
  const double beta = first ? 0.0
                      : flexible ? (S[S_PT] != 0.0 ? -S[S_ZT] / S[S_PT] : 0.0)
                                 : (S[S_RZ] == 0.0 ? 0.0 : S[S_RZNEW] / S[S_RZ]);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    p[t] = first ? z[t] : fma(beta, p[t], z[t]);
}

__global__ void copy_scalar_kernel(double* S, int dst, int src) { S[dst] = S[src]; }

// default power-iteration start vector: splitmix64 counter generator (synth.splitmix_uniform)
// indexed by the GLOBAL dof: a slab's vector is the slice of the one-GPU vector (replicated
// interface planes identical on both ranks); nodes / nodes_g local / global nodes per
// component, off = first global node of the slab
__global__ void splitmix_kernel(double* __restrict__ v, int64_t n, unsigned long long seed, int64_t nodes,
                                int64_t nodes_g, int64_t off) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tg = (t / nodes) * nodes_g + off + t % nodes;
    unsigned long long z = seed + (unsigned long long)(tg + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    v[t] = 2.0 * (double)(z >> 11) * 0x1.0p-53 - 1.0;
  }
}

int ensure_red(elas_op* op) {
  if (!op->red) {
    CK(cudaMalloc(&op->red, sizeof(double) * (RED_BLOCKS + S_COUNT + 1)), "cudaMalloc (reduction scratch)");
    CK(cudaMemset(op->red, 0, sizeof(double) * (RED_BLOCKS + S_COUNT + 1)), "cudaMemset (reduction scratch)");
  }
  return ELAS_OK;
}

int read_scalar(elas_op* op, int slot, double* out) {
  CK(cudaMemcpyAsync(out, op->red + RED_BLOCKS + slot, sizeof(double), cudaMemcpyDeviceToHost, op->stream),
     "cudaMemcpyAsync (scalar)");
  CK(cudaStreamSynchronize(op->stream), "cudaStreamSynchronize");
  return ELAS_OK;
}

int ensure_dinv(elas_op* op);

}  // namespace

void free_solver_state(elas_op* op) {
  cudaFree(op->dinv);
  cudaFree(op->red);
  cudaFree(op->work);
  op->dinv = op->red = op->work = nullptr;
}

}  // namespace elas


namespace elas {
namespace {

int diag_raw(elas_op* op, double* d) {
  const Slab& s = op->slab;
  const int p = op->p, q = op->q, n = p + 1;
  const size_t smem = sizeof(double) * (size_t)(5 * q * n + 3 * (q * q * q + q * q * n + q * n * n + n * n * n));
  // a per-device function attribute: set on the op's (current) device on every call (setup path)
  CK(cudaFuncSetAttribute(diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "cudaFuncSetAttribute");
  diag_init_kernel<<<grid_for(3 * s.nodes), 256, 0, op->stream>>>(s, d);
  const int64_t ne = (int64_t)s.nx * s.ny * s.nz;
  const double* gauss = op->tab + tables_gauss_offset(p, q, fold_table_size(p, q));
  if (ne > 0) diag_kernel<<<(unsigned)ne, 128, smem, op->stream>>>(p, q, op->qlayout, s, op->qd, op->rr, op->tab, gauss, op->cc, d);
  CK(cudaGetLastError(), "diagonal kernels");
  return exchange_planes(op, d);
}

int ensure_dinv(elas_op* op) {
  if (op->dinv) return ELAS_OK;
  const int64_t n = 3 * op->slab.nodes;
  double* d = nullptr;
  CK(cudaMalloc(&d, sizeof(double) * n), "cudaMalloc (diagonal)");
  int rc = diag_raw(op, d);
  if (rc) { cudaFree(d); return rc; }
  inv_kernel<<<grid_for(n), 256, 0, op->stream>>>(d, d, n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { cudaFree(d); return fail(e, "inverse diagonal"); }
  op->dinv = d;
  return ELAS_OK;
}

bool solver_ok(const elas_op* op, const char* who) {
  if (op->nranks != 1 && !op->comm) {
    set_error(std::string(who) + ": distributed solvers need the NCCL slab mode (external-exchange ops "
              "cannot reduce dots)");
    return false;
  }
  return true;
}

}  // namespace

// x <- x + p_k(D^{-1}A) D^{-1}(b - A x); x_zero: treat x as 0 on entry (preconditioner form)
int cheb_run(elas_cheb* ch, const double* b, double* x, bool x_zero) {
  elas_op* op = ch->op;
  const int64_t n = 3 * op->slab.nodes;
  double* r = ch->buf;
  double* dv = r + n;
  double* t = dv + n;
  cudaStream_t st = op->stream;
  const double lo = ch->alpha * ch->lam_max, hi = ch->beta * ch->lam_max;
  const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo);
  int rc;
  if (!x_zero) {
    if ((rc = elas_apply(op, x, t))) return rc;
  }
  cheb_start_kernel<<<grid_for(n), 256, 0, st>>>(b, x_zero ? nullptr : t, op->dinv, r, dv, x, 1.0 / theta,
                                                 x_zero ? 1 : 0, n);
  CK(cudaGetLastError(), "chebyshev start kernel");
  if (ch->order == 1) return ELAS_OK;
  const double sigma = theta / delta;
  double rho = 1.0 / sigma;
  for (int k = 2; k <= ch->order; ++k) {
    if ((rc = elas_apply(op, dv, t))) return rc;
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    cheb_step_kernel<<<grid_for(n), 256, 0, st>>>(t, op->dinv, r, dv, x, rho_new * rho, 2.0 * rho_new / delta, n);
    CK(cudaGetLastError(), "chebyshev step kernel");
    rho = rho_new;
  }
  return ELAS_OK;
}

int pcg_core(elas_op* op, int kind, const PrecondFn& M, const double* b, double* x, double rtol, int maxit,
             bool check, elas_solve_report* rep, double* history, bool flexible) {
  int rc;
  if ((rc = ensure_red(op))) return rc;
  if (kind == ELAS_PC_JACOBI && (rc = ensure_dinv(op))) return rc;
  const int64_t n = 3 * op->slab.nodes;
  if (!op->work) CK(cudaMalloc(&op->work, sizeof(double) * 4 * n), "cudaMalloc (pcg work vectors)");
  double* r = op->work;
  double* z = r + n;
  double* p = z + n;
  double* t = p + n;
  cudaStream_t st = op->stream;
  const int g = grid_for(n);
  double* S = op->red + RED_BLOCKS;
  const bool fused_z = kind != PC_CALLBACK;
  // x = 0, r = b, z = M r
  CK(cudaMemsetAsync(x, 0, sizeof(double) * n, st), "cudaMemsetAsync");
  CK(cudaMemcpyAsync(r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "cudaMemcpyAsync");
  if (kind == PC_CALLBACK) {
    if ((rc = M(r, z))) return rc;
  } else if (kind == ELAS_PC_JACOBI) {
    scale_kernel<<<g, 256, 0, st>>>(z, op->dinv, r, n);
  } else {
    CK(cudaMemcpyAsync(z, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "cudaMemcpyAsync");
  }
  CK(cudaGetLastError(), "preconditioner kernel");
  if ((rc = dot(op, r, z, S_RZ))) return rc;
  double rz0 = 1.0;
  if (check) {
    if ((rc = read_scalar(op, S_RZ, &rz0))) return rc;
    if (rz0 < 0.0 || !std::isfinite(rz0)) { set_error("elas_pcg: preconditioner not positive definite"); return ELAS_EINVAL; }
  }
  int it = 0;
  double rel = rz0 > 0.0 ? 1.0 : 0.0;
  if (history) history[0] = rel;
  if (rz0 > 0.0) {
    pcg_direction_kernel<<<g, 256, 0, st>>>(p, z, S, n, 1, 0);
    while (it < maxit) {
      if ((rc = elas_apply(op, p, t))) return rc;
      if ((rc = dot(op, p, t, S_PT))) return rc;
      pcg_update_kernel<<<g, 256, 0, st>>>(x, r, fused_z ? z : nullptr, p, t,
                                           kind == ELAS_PC_JACOBI ? op->dinv : nullptr, S, n);
      CK(cudaGetLastError(), "pcg update kernel");
      if (!fused_z && (rc = M(r, z))) return rc;
      if ((rc = dot(op, r, z, S_RZNEW))) return rc;
      if (flexible && (rc = dot(op, z, t, S_ZT))) return rc;
      ++it;
      if (check) {
        double rz = 0.0;
        if ((rc = read_scalar(op, S_RZNEW, &rz))) return rc;
        rel = std::sqrt(rz > 0.0 ? rz / rz0 : 0.0);
        if (history) history[it] = rel;
        if (rel <= rtol) break;
      }
      pcg_direction_kernel<<<g, 256, 0, st>>>(p, z, S, n, 0, flexible ? 1 : 0);
      copy_scalar_kernel<<<1, 1, 0, st>>>(S, S_RZ, S_RZNEW);
      CK(cudaGetLastError(), "pcg direction kernels");
    }
  }
  if (rep) {
    rep->iterations = it;
    rep->rel_residual = check ? rel : -1.0;
    rep->converged = (check && rel <= rtol) ? 1 : 0;
  }
  return ELAS_OK;
}

}  // namespace elas

using elas::Slab;

extern "C" {

int elas_diagonal(elas_op* op, double* d) {
  if (!op || !d) { elas::set_error("elas_diagonal: NULL argument"); return ELAS_EINVAL; }
  if ((uintptr_t)d & 7u) { elas::set_error("elas_diagonal: d must be 8-byte aligned"); return ELAS_EINVAL; }
  return elas::diag_raw(op, d);
}

elas_cheb* elas_cheb_create(elas_op* op, int order, double alpha, double beta, int power_iters, const double* v0,
                            unsigned long long seed) {
  if (!op) { elas::set_error("elas_cheb_create: NULL op"); return nullptr; }
  if (!elas::solver_ok(op, "elas_cheb_create")) return nullptr;
  if (order < 1 || power_iters < 1 || !(alpha > 0.0) || !(beta > alpha) || !std::isfinite(beta)) {
    elas::set_error("elas_cheb_create: need order >= 1, power_iters >= 1, 0 < alpha < beta");
    return nullptr;
  }
  if (elas::ensure_dinv(op) || elas::ensure_red(op)) return nullptr;
  const int64_t n = 3 * op->slab.nodes;
  elas_cheb* ch = new elas_cheb();
  ch->op = op;
  ch->order = order;
  ch->alpha = alpha;
  ch->beta = beta;
  auto bail = [&](cudaError_t e, const char* what) -> elas_cheb* {
    if (e != cudaSuccess) elas::set_error(std::string(what) + ": " + cudaGetErrorString(e));
    cudaFree(ch->buf);
    delete ch;
    return nullptr;
  };
  cudaError_t e = cudaMalloc(&ch->buf, sizeof(double) * 3 * n);
  if (e != cudaSuccess) return bail(e, "cudaMalloc (chebyshev work vectors)");
  // power iteration on D^{-1} A: v <- v/|v|; w = D^{-1} A v; lam = v.w; v <- w/|w|
  double* v = ch->buf;
  double* w = v + n;
  double* t = w + n;
  cudaStream_t st = op->stream;
  const int g = elas::grid_for(n);
  double* S = op->red + elas::RED_BLOCKS;
  if (v0) e = cudaMemcpyAsync(w, v0, sizeof(double) * n, cudaMemcpyDeviceToDevice, st);
  else {
    const elas::Slab& sl = op->slab;
    const int64_t plane = (int64_t)sl.Nx * sl.Ny;
    const int64_t nodes_g = plane * ((int64_t)op->nz_global * op->p + 1);
    elas::splitmix_kernel<<<g, 256, 0, st>>>(w, n, seed, sl.nodes, nodes_g, plane * (int64_t)op->ez0 * op->p);
  }
  if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) return bail(e, "power iteration start vector");
  if (elas::dot(op, w, w, elas::S_NRM)) return bail(cudaSuccess, "");
  elas::normalize_kernel<<<g, 256, 0, st>>>(v, w, S + elas::S_NRM, n);
  for (int it = 0; it < power_iters; ++it) {
    if (elas_apply(op, v, t)) return bail(cudaSuccess, "");
    elas::scale_kernel<<<g, 256, 0, st>>>(w, op->dinv, t, n);
    if (elas::dot(op, v, w, elas::S_LAM) || elas::dot(op, w, w, elas::S_NRM))
      return bail(cudaSuccess, "");
    elas::normalize_kernel<<<g, 256, 0, st>>>(v, w, S + elas::S_NRM, n);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return bail(e, "power iteration kernels");
  double lam = 0.0;
  if (elas::read_scalar(op, elas::S_LAM, &lam)) return bail(cudaSuccess, "");
  if (!(lam > 0.0) || !std::isfinite(lam)) {
    elas::set_error("elas_cheb_create: power iteration gave a non-positive estimate (zero operator?)");
    return bail(cudaSuccess, "");
  }
  ch->lam_max = 1.1 * lam;
  return ch;
}

double elas_cheb_lambda_max(const elas_cheb* ch) { return ch ? ch->lam_max : -1.0; }

int elas_cheb_apply(elas_cheb* ch, const double* b, double* x) {
  if (!ch || !b || !x) { elas::set_error("elas_cheb_apply: NULL argument"); return ELAS_EINVAL; }
  if (b == x) { elas::set_error("elas_cheb_apply: b and x must not alias"); return ELAS_EINVAL; }
  return elas::cheb_run(ch, b, x, false);
}

void elas_cheb_destroy(elas_cheb* ch) {
  if (!ch) return;
  cudaStreamSynchronize(ch->op->stream);
  cudaFree(ch->buf);
  delete ch;
}

int elas_pcg(elas_op* op, int precond, elas_cheb* cheb, const double* b, double* x, double rtol, int maxit,
             elas_solve_report* rep, double* history) {
  if (!op || !b || !x) { elas::set_error("elas_pcg: NULL argument"); return ELAS_EINVAL; }
  if (!elas::solver_ok(op, "elas_pcg")) return ELAS_EINVAL;
  if (precond < ELAS_PC_NONE || precond > ELAS_PC_CHEBYSHEV ||
      (precond == ELAS_PC_CHEBYSHEV && (!cheb || cheb->op->slab.nodes != op->slab.nodes ||
                                        cheb->op->stream != op->stream))) {
    elas::set_error("elas_pcg: unknown preconditioner, or a Chebyshev preconditioner whose operator has another "
                    "vector length or stream");
    return ELAS_EINVAL;
  }
  if (b == x || maxit < 0 || !(rtol >= 0.0)) { elas::set_error("elas_pcg: need b != x, maxit >= 0, rtol >= 0"); return ELAS_EINVAL; }
  if (precond == ELAS_PC_CHEBYSHEV)
    return elas::pcg_core(op, elas::PC_CALLBACK,
                          [cheb](const double* r, double* z) { return elas::cheb_run(cheb, r, z, true); }, b, x,
                          rtol, maxit, true, rep, history);
  return elas::pcg_core(op, precond, elas::PrecondFn(), b, x, rtol, maxit, true, rep, history);
}

int elas_dot(elas_op* op, const double* a, const double* b, double* result) {
  if (!op || !a || !b || !result) { elas::set_error("elas_dot: NULL argument"); return ELAS_EINVAL; }
  int rc;
  if ((rc = elas::ensure_red(op))) return rc;
  if ((rc = elas::dot(op, a, b, elas::S_DOT))) return rc;
  return elas::read_scalar(op, elas::S_DOT, result);
}

}  // extern "C"
