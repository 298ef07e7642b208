// Setup and small per-apply kernels:
//  * qdata kernel (the "assembly" phase of partial assembly; Alg. 1 inputs
//    geom.J(p,e), ipWeights[p], lambda(p,e), mu(p,e); Table 3 "Assembly" column):
//      J_mk = d x_m / d xi_k of the trilinear map (8 vertices) at each Gauss point,
//      det J (> 0, else ELAS_EGEOM), A = J^{-1}, W = w_a w_b w_c det J,
//      stored:  A~ = sqrt(mu_e W) A  (9 doubles per point)  and  r_e = lambda_e / mu_e.
//    With H = G A~ and sigma~ = r tr(H) I + H + H^T,  sigma~ A~^T = W sigma A^T exactly
//    (DESIGN.md section 5): 9 doubles per point is the minimal stored form.
//    Layout qd[e][a1][f][L], L = a3 + q a2 (the x-line index of the apply kernel), so the
//    threads of one warp read consecutive doubles.
//  * init kernel: y = (I - Z) x  (0 on free dofs, x on Dirichlet dofs) before the atomics.
//  * plane-add kernel: y_plane += halo on free dofs (multi-GPU interface sum, P^T of
//    PAPER.md:169).
#include <algorithm>

#include "elas_internal.h"

namespace elas {

namespace {

__device__ __forceinline__ bool constrained_node(int I, int J, int K, const Slab& s) {
  const uint32_t f = s.faces;
  return ((f & ELAS_FACE_XMIN) && I == 0) || ((f & ELAS_FACE_XMAX) && I == s.Nx - 1) ||
         ((f & ELAS_FACE_YMIN) && J == 0) || ((f & ELAS_FACE_YMAX) && J == s.Ny - 1) ||
         ((f & ELAS_FACE_ZMIN) && K == 0) || ((f & ELAS_FACE_ZMAX) && K == s.Nz - 1);
}

struct QParams {
  double g[16];
  double w[16];
};

__global__ void qdata_kernel(int q, int layout, Slab s, const double* __restrict__ V, const double* __restrict__ lam,
                             const double* __restrict__ mu, QParams qp, double* __restrict__ qd,
                             double* __restrict__ rr, int* __restrict__ bad, int64_t total) {
  const int q3 = q * q * q;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / q3;
    const int pt = (int)(t % q3);
    const int a1 = pt % q, a2 = (pt / q) % q, a3 = pt / (q * q);
    const int ex = (int)(e % s.nx), ey = (int)((e / s.nx) % s.ny), ez = (int)(e / ((int64_t)s.nx * s.ny));
    const double xi[3] = {qp.g[a1], qp.g[a2], qp.g[a3]};
    double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int c = 0; c < 2; ++c)
      for (int b = 0; b < 2; ++b)
        for (int a = 0; a < 2; ++a) {
          const int64_t v = ((int64_t)(ez + c) * (s.ny + 1) + (ey + b)) * (s.nx + 1) + (ex + a);
          const double h0 = a ? xi[0] : 1.0 - xi[0], d0 = a ? 1.0 : -1.0;
          const double h1 = b ? xi[1] : 1.0 - xi[1], d1 = b ? 1.0 : -1.0;
          const double h2 = c ? xi[2] : 1.0 - xi[2], d2 = c ? 1.0 : -1.0;
          const double dN[3] = {d0 * h1 * h2, h0 * d1 * h2, h0 * h1 * d2};
          for (int m = 0; m < 3; ++m) {
            const double X = V[v * 3 + m];
            for (int k = 0; k < 3; ++k) J[m][k] = fma(X, dN[k], J[m][k]);
          }
        }
    // adjugate / determinant
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
    if (!(det > 0.0)) {
      atomicExch(bad, 1);
      continue;
    }
    const double W = qp.w[a1] * qp.w[a2] * qp.w[a3] * det;
    const double sc = sqrt(mu[e] * W) / det;   // A~ = sqrt(mu W) J^{-1} = sqrt(mu W) adj / det
    if (layout == QD_LAYOUT_OTF || layout == QD_LAYOUT_OTF32) {   // geometry on the fly: det check above,
      if (pt == 0) {                   // the Jacobian polynomial coefficients once per element
        double Xv[2][2][2][3];
        for (int c = 0; c < 2; ++c)
          for (int b = 0; b < 2; ++b)
            for (int a = 0; a < 2; ++a) {
              const int64_t v = ((int64_t)(ez + c) * (s.ny + 1) + (ey + b)) * (s.nx + 1) + (ex + a);
              for (int m = 0; m < 3; ++m) Xv[a][b][c][m] = V[v * 3 + m];
            }
        double ow[GEO_WORDS];
        double* o = ow;
        for (int m = 0; m < 3; ++m) {
          // d/dxi1: differences along a, bilinear in (xi2 = b, xi3 = c)
          const double d00 = Xv[1][0][0][m] - Xv[0][0][0][m], d10 = Xv[1][1][0][m] - Xv[0][1][0][m];
          const double d01 = Xv[1][0][1][m] - Xv[0][0][1][m], d11 = Xv[1][1][1][m] - Xv[0][1][1][m];
          o[0 + m] = d00; o[3 + m] = d10 - d00; o[6 + m] = d01 - d00; o[9 + m] = d11 - d10 - d01 + d00;
          // d/dxi2: differences along b, bilinear in (xi1 = a, xi3 = c)
          const double g00 = Xv[0][1][0][m] - Xv[0][0][0][m], g10 = Xv[1][1][0][m] - Xv[1][0][0][m];
          const double g01 = Xv[0][1][1][m] - Xv[0][0][1][m], g11 = Xv[1][1][1][m] - Xv[1][0][1][m];
          o[12 + m] = g00; o[15 + m] = g10 - g00; o[18 + m] = g01 - g00; o[21 + m] = g11 - g10 - g01 + g00;
          // d/dxi3: differences along c, bilinear in (xi1 = a, xi2 = b)
          const double h00 = Xv[0][0][1][m] - Xv[0][0][0][m], h10 = Xv[1][0][1][m] - Xv[1][0][0][m];
          const double h01 = Xv[0][1][1][m] - Xv[0][1][0][m], h11 = Xv[1][1][1][m] - Xv[1][1][0][m];
          o[24 + m] = h00; o[27 + m] = h10 - h00; o[30 + m] = h01 - h00; o[33 + m] = h11 - h10 - h01 + h00;
        }
        o[36] = sqrt(mu[e]);
        o[37] = o[38] = o[39] = 0.0;
        for (int w = 0; w < GEO_WORDS; ++w) {
          if (layout == QD_LAYOUT_OTF) qd[e * (int64_t)GEO_WORDS + w] = ow[w];
          else qd[(e >> 5) * (int64_t)(32 * GEO_WORDS) + w * 32 + (e & 31)] = ow[w];
        }
      }
    } else if (layout == QD_LAYOUT_E32) {
      double* out = qd + (e >> 5) * (int64_t)(32 * 9 * q3) + (int64_t)pt * 9 * 32 + (e & 31);
      for (int d = 0; d < 3; ++d)
        for (int m = 0; m < 3; ++m) out[(3 * d + m) * 32] = sc * adj[d][m];
    } else if (layout == QD_LAYOUT_TC6) {
      // fragment order of apply_tc_kernel (q = 8): 32 lanes contiguous per (slice, r, f)
      const int sl = a1 >> 1, r = 2 * (a1 & 1) + (a3 & 1), lane = 4 * a2 + (a3 >> 1);
      double* out = qd + e * (int64_t)(9 * q3) + (int64_t)((sl * 4 + r) * 9) * 32 + lane;
      for (int d = 0; d < 3; ++d)
        for (int m = 0; m < 3; ++m) out[(3 * d + m) * 32] = sc * adj[d][m];
    } else if (layout == QD_LAYOUT_LINES_F32) {   // mixed precision: the same values rounded to FP32
      const int L = a3 + q * a2;
      float* out = reinterpret_cast<float*>(qd) + e * (int64_t)((9 * q3 + 3) & ~3) +
                   (int64_t)a1 * 9 * q * q + L;
      for (int d = 0; d < 3; ++d)
        for (int m = 0; m < 3; ++m) out[(3 * d + m) * q * q] = (float)(sc * adj[d][m]);
    } else {
      const int L = a3 + q * a2;
      double* out = qd + e * (int64_t)qd_stride_lines(q) + (int64_t)a1 * 9 * q * q + L;
      for (int d = 0; d < 3; ++d)
        for (int m = 0; m < 3; ++m) out[(3 * d + m) * q * q] = sc * adj[d][m];
    }
    if (pt == 0) rr[e] = lam[e] / mu[e];
  }
}



__global__ void plane_add_kernel(Slab s, int K, double* __restrict__ y, const double* __restrict__ halo) {
  const int64_t plane = (int64_t)s.Nx * s.Ny;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 3 * plane; t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t / plane);
    const int64_t pidx = t % plane;
    const int I = (int)(pidx % s.Nx), J = (int)(pidx / s.Nx);
    if (s.faces && constrained_node(I, J, K, s)) continue;
    double* dst = y + c * s.nodes + (int64_t)K * plane + pidx;
    ELAS_DCHECK(K >= 0 && K < s.Nz && c * s.nodes + (int64_t)K * plane + pidx < 3 * s.nodes);
    *dst = *dst + halo[t];
  }
}

// debug-build self-test: one deliberately failed check (elas_debug_checks(..., selftest = 1))
__global__ void dcheck_selftest_kernel(int v) { ELAS_DCHECK(v == 0); }

__global__ void wait_flag_kernel(const unsigned long long* flag, unsigned long long target) {
  unsigned long long v;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= target) break;
    __nanosleep(128);
  }
}

__global__ void signal_flag_kernel(unsigned long long* flag, unsigned long long value) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
}

int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = 148 * 32;
  return (int)(g < cap ? (g > 0 ? g : 1) : cap);
}

}  // namespace

cudaError_t launch_qdata(int p, int q, int layout, const Slab& s, const double* verts, const double* lam,
                         const double* mu, const double* gpts, const double* gw, double* qd,
                         double* rr, int* bad, cudaStream_t st) {
  (void)p;
  QParams qp{};
  for (int a = 0; a < q; ++a) {
    qp.g[a] = gpts[a];
    qp.w[a] = gw[a];
  }
  const int64_t total = (int64_t)s.nx * s.ny * s.nz * q * q * q;
  qdata_kernel<<<grid_for(total, 256), 256, 0, st>>>(q, layout, s, verts, lam, mu, qp, qd, rr, bad, total);
  return cudaGetLastError();
}

// y = (I - Z) x on node planes [K0, K1): a memset of the planes plus a copy of x on the
// constrained face nodes only (blockIdx.y = face); the general init_kernel computed node
// coordinates for every dof (64-bit divisions) and cost ~25 % of an apply on Dirichlet meshes.
// add = 0: y = x on the constrained face nodes; add = 1: y += x, each node once (a node on several
// constrained faces is handled by the lowest-numbered one)
__global__ void face_copy_kernel(Slab s, int K0, int K1, const double* __restrict__ x, double* __restrict__ y,
                                 int add) {
  const int face = blockIdx.y;
  if (!(s.faces & (1u << face))) return;
  const int axis = face >> 1, hi = face & 1;
  // the two free axes of the face, K clipped to [K0, K1)
  const int n0 = axis == 0 ? s.Ny : s.Nx;
  const int k0 = axis == 2 ? 0 : K0, k1 = axis == 2 ? 1 : K1;
  const int n1 = axis == 2 ? s.Ny : (k1 - k0);
  if (axis == 2) {   // z face: only its own plane, if inside [K0, K1)
    const int K = hi ? s.Nz - 1 : 0;
    if (K < K0 || K >= K1) return;
  }
  const int64_t per_c = (int64_t)n0 * n1;
  const int64_t plane = (int64_t)s.Nx * s.Ny;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 3 * per_c; t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t / per_c);
    const int64_t r = t - c * per_c;
    const int a = (int)(r % n0), b = (int)(r / n0);
    int I, J, K;
    if (axis == 0) { I = hi ? s.Nx - 1 : 0; J = a; K = k0 + b; }
    else if (axis == 1) { I = a; J = hi ? s.Ny - 1 : 0; K = k0 + b; }
    else { I = a; J = b; K = hi ? s.Nz - 1 : 0; }
    const int64_t idx = c * s.nodes + (int64_t)K * plane + (int64_t)J * s.Nx + I;
    if (!add) {
      y[idx] = x[idx];
    } else {
      bool lower = false;   // on a lower-numbered constrained face?
      for (int f2 = 0; f2 < face; ++f2) {
        if (!(s.faces & (1u << f2))) continue;
        const int ax2 = f2 >> 1, hi2 = f2 & 1;
        const int v = ax2 == 0 ? I : ax2 == 1 ? J : K;
        const int vmax = ax2 == 0 ? s.Nx - 1 : ax2 == 1 ? s.Ny - 1 : s.Nz - 1;
        if (v == (hi2 ? vmax : 0)) lower = true;
      }
      if (!lower) y[idx] += x[idx];
    }
  }
}

cudaError_t launch_init(const Slab& s, const double* x, double* y, cudaStream_t st) {
  return launch_init_planes(s, 0, s.Nz, x, y, st);
}

cudaError_t launch_init_planes(const Slab& s, int K0, int K1, const double* x, double* y, cudaStream_t st) {
  if (K1 <= K0) return cudaSuccess;
  const int64_t plane = (int64_t)s.Nx * s.Ny;
  cudaError_t e;
  if (K0 == 0 && K1 == s.Nz) {
    e = cudaMemsetAsync(y, 0, sizeof(double) * 3 * (size_t)s.nodes, st);
  } else {
    e = cudaSuccess;
    for (int c = 0; c < 3 && e == cudaSuccess; ++c)
      e = cudaMemsetAsync(y + c * s.nodes + (int64_t)K0 * plane, 0, sizeof(double) * (size_t)(K1 - K0) * plane, st);
  }
  if (e != cudaSuccess || !s.faces) return e;
  const int64_t maxface = 3 * (int64_t)std::max(std::max(s.Nx, s.Ny), K1 - K0) * std::max(std::max(s.Ny, s.Nx), K1 - K0);
  face_copy_kernel<<<dim3((unsigned)grid_for(maxface, 256), 6), 256, 0, st>>>(s, K0, K1, x, y, 0);
  return cudaGetLastError();
}

cudaError_t launch_face_copy(const Slab& s, const double* x, double* y, cudaStream_t st) {
  if (!s.faces) return cudaSuccess;
  const int64_t m = std::max(std::max(s.Nx, s.Ny), s.Nz);
  face_copy_kernel<<<dim3((unsigned)grid_for(3 * m * m, 256), 6), 256, 0, st>>>(s, 0, s.Nz, x, y, 0);
  return cudaGetLastError();
}

cudaError_t launch_face_add(const Slab& s, const double* x, double* y, cudaStream_t st) {
  if (!s.faces) return cudaSuccess;
  const int64_t m = std::max(std::max(s.Nx, s.Ny), s.Nz);
  face_copy_kernel<<<dim3((unsigned)grid_for(3 * m * m, 256), 6), 256, 0, st>>>(s, 0, s.Nz, x, y, 1);
  return cudaGetLastError();
}

cudaError_t launch_plane_add(const Slab& s, int which_plane, double* y, const double* halo, cudaStream_t st) {
  const int64_t n = 3 * (int64_t)s.Nx * s.Ny;
  plane_add_kernel<<<grid_for(n, 256), 256, 0, st>>>(s, which_plane, y, halo);
  return cudaGetLastError();
}

cudaError_t launch_wait_flag(const unsigned long long* flag, unsigned long long target, cudaStream_t st) {
  if (target == 0) return cudaSuccess;   // nothing to wait for (first exchange)
  wait_flag_kernel<<<1, 1, 0, st>>>(flag, target);
  return cudaGetLastError();
}

cudaError_t launch_signal_flag(unsigned long long* flag, unsigned long long value, cudaStream_t st) {
  signal_flag_kernel<<<1, 1, 0, st>>>(flag, value);
  return cudaGetLastError();
}

cudaError_t launch_dcheck_selftest(cudaStream_t st) {
  dcheck_selftest_kernel<<<1, 1, 0, st>>>(1);
  return cudaGetLastError();
}

}  // namespace elas

ELAS_DCHECK_READER(dcheck_setup)
