// Host-side 1D tables for the sum-factorised kernels: the factors B_1D, D_1D of
// G_xi = D_1D (x) B_1D (x) B_1D (Sec. 2.2.3) on the reference interval [0,1].
//
//  * GLL nodes (reading R2): Newton's method on (1 - t^2) P_p'(t) = 0 started from
//    the Chebyshev-Gauss-Lobatto points, Legendre values by the three-term recurrence;
//    symmetrised so that xi_{p-i} = 1 - xi_i and the midpoint is exactly 1/2.
//  * Gauss-Legendre rule with q points (reading R3): Newton on P_q(t) = 0, weights
//    2 / ((1 - t^2) P_q'(t)^2), mapped to [0,1] (weights halved, sum 1).
//  * Lagrange cardinal functions in BARYCENTRIC form:
//      l_i(t) = (w_i / (t - xi_i)) / sum_j (w_j / (t - xi_j)),  w_i = 1 / prod_{j!=i} (xi_i - xi_j)
//      l_i'(t) = l_i(t) * sum_{j != i} 1 / (t - xi_j)            (t not a node)
//    and, where a point coincides with a node xi_k, the differentiation-matrix row
//      l_i'(xi_k) = (w_i / w_k) / (xi_k - xi_i) (i != k),  l_k'(xi_k) = -sum_{i != k} l_i'(xi_k).
// This file shares nothing with oracle/ (which uses numpy roots and the product formula).
#include <cmath>
#include <vector>

#include "elas_internal.h"

namespace elas {
namespace {

// P_n(t) and P_n'(t) by the three-term recurrence.
void legendre(int n, double t, double* P, double* dP) {
  double p0 = 1.0, p1 = t;
  if (n == 0) { *P = 1.0; *dP = 0.0; return; }
  for (int k = 2; k <= n; ++k) {
    double p2 = ((2.0 * k - 1.0) * t * p1 - (k - 1.0) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  *P = p1;
  // P_n'(t) = n (t P_n - P_{n-1}) / (t^2 - 1)   (t != +-1 for interior roots)
  *dP = n * (t * p1 - p0) / (t * t - 1.0);
}

void gll_nodes(int p, double* x) {
  // roots t of P_p'(t) in (-1, 1); P_p'' from the Legendre ODE:
  // (1 - t^2) P'' = 2 t P' - p (p + 1) P
  std::vector<double> t(p + 1);
  t[0] = -1.0;
  t[p] = 1.0;
  for (int i = 1; i < p; ++i) {
    double s = -std::cos(M_PI * i / p);
    for (int it = 0; it < 100; ++it) {
      double P, dP;
      legendre(p, s, &P, &dP);
      double d2P = (2.0 * s * dP - p * (p + 1.0) * P) / (1.0 - s * s);
      double ds = dP / d2P;
      s -= ds;
      if (std::fabs(ds) < 1e-17) break;
    }
    t[i] = s;
  }
  for (int i = 0; i <= p; ++i) x[i] = 0.5 * (1.0 + t[i]);
  // symmetrise: lower half kept, upper half mirrored, exact midpoint
  for (int i = 0; i <= p / 2; ++i) {
    double lo = 0.5 * (x[i] + (1.0 - x[p - i]));
    x[i] = lo;
    x[p - i] = 1.0 - lo;
  }
  if (p % 2 == 0) x[p / 2] = 0.5;
  x[0] = 0.0;
  x[p] = 1.0;
}

void gauss_legendre(int q, double* g, double* w) {
  for (int i = 0; i < q; ++i) {
    double s = -std::cos(M_PI * (i + 0.75) / (q + 0.5));
    double P = 0, dP = 1;
    for (int it = 0; it < 100; ++it) {
      legendre(q, s, &P, &dP);
      double ds = P / dP;
      s -= ds;
      if (std::fabs(ds) < 1e-17) break;
    }
    legendre(q, s, &P, &dP);
    g[i] = s;
    w[i] = 2.0 / ((1.0 - s * s) * dP * dP);
  }
  for (int i = 0; i < q / 2; ++i) {  // symmetrise
    double s = 0.5 * (g[q - 1 - i] - g[i]);
    double ww = 0.5 * (w[i] + w[q - 1 - i]);
    g[i] = -s;
    g[q - 1 - i] = s;
    w[i] = w[q - 1 - i] = ww;
  }
  if (q % 2 == 1) g[q / 2] = 0.0;
  for (int i = 0; i < q; ++i) {
    g[i] = 0.5 * (1.0 + g[i]);
    w[i] = 0.5 * w[i];
  }
  for (int i = 0; i < q / 2; ++i) g[q - 1 - i] = 1.0 - g[i];
}

}  // namespace

int host_tables(int p, int q, double* nodes, double* points, double* weights, double* B, double* D) {
  if (p < 1 || p > 8 || q < 1 || q > 16) return ELAS_EINVAL;
  const int n = p + 1;
  std::vector<double> xi(n), g(q), w(q), bw(n);
  gll_nodes(p, xi.data());
  gauss_legendre(q, g.data(), w.data());
  for (int i = 0; i < n; ++i) {
    double prod = 1.0;
    for (int j = 0; j < n; ++j)
      if (j != i) prod *= (xi[i] - xi[j]);
    bw[i] = 1.0 / prod;
  }
  for (int a = 0; a < q; ++a) {
    const double t = g[a];
    int hit = -1;
    for (int k = 0; k < n; ++k)
      if (t == xi[k]) hit = k;
    if (hit >= 0) {
      double diag = 0.0;
      for (int i = 0; i < n; ++i) {
        if (B) B[a * n + i] = (i == hit) ? 1.0 : 0.0;
        if (i != hit) {
          double d = (bw[i] / bw[hit]) / (xi[hit] - xi[i]);
          if (D) D[a * n + i] = d;
          diag -= d;
        }
      }
      if (D) D[a * n + hit] = diag;
      continue;
    }
    double denom = 0.0;
    for (int j = 0; j < n; ++j) denom += bw[j] / (t - xi[j]);
    for (int i = 0; i < n; ++i) {
      double li = (bw[i] / (t - xi[i])) / denom;
      if (B) B[a * n + i] = li;
      double s = 0.0;
      for (int j = 0; j < n; ++j)
        if (j != i) s += 1.0 / (t - xi[j]);
      if (D) D[a * n + i] = li * s;
    }
  }
  if (nodes)
    for (int i = 0; i < n; ++i) nodes[i] = xi[i];
  if (points)
    for (int a = 0; a < q; ++a) points[a] = g[a];
  if (weights)
    for (int a = 0; a < q; ++a) weights[a] = w[a];
  return ELAS_OK;
}

// Even-odd folded form of one q x n table T (B: parity +1, D: parity -1), DESIGN.md section 6.
// GLL nodes and Gauss points are symmetric about 1/2, so T[q-1-a][n-1-i] = s T[a][i].  With
// u+_i = u_i + u_{n-1-i}, u-_i = u_i - u_{n-1-i} (i < n/2) the forward contraction is
//   E_a = sum_i FE[a][i] u+_i (+ FE[a][n/2] u_mid),  O_a = sum_i FO[a][i] u-_i,
//   (T u)_a = E_a + O_a,  (T u)_{q-1-a} = s (E_a - O_a)                 (a < (q+1)/2)
// and the transposed one the same with the roles of points and nodes swapped (BE, BO).
// Layout (fold_table_size doubles): FE[qe][ne] | FO[qe][nh] | BE[ne][qe] | BO[ne][qh],
// ne = (n+1)/2, nh = n/2, qe = (q+1)/2, qh = q/2.
int fold_table_size(int p, int q) { return ((q + 1) / 2) * (p + 1) + ((p + 2) / 2) * q; }

void host_fold_table(int p, int q, const double* T, double* out) {
  const int n = p + 1, ne = (n + 1) / 2, nh = n / 2, qe = (q + 1) / 2, qh = q / 2;
  double* FE = out;
  double* FO = FE + qe * ne;
  double* BE = FE + qe * n;
  double* BO = BE + ne * qe;
  for (int a = 0; a < qe; ++a) {
    for (int i = 0; i < nh; ++i) {
      FE[a * ne + i] = 0.5 * (T[a * n + i] + T[a * n + n - 1 - i]);
      FO[a * nh + i] = 0.5 * (T[a * n + i] - T[a * n + n - 1 - i]);
    }
    if (n & 1) FE[a * ne + nh] = T[a * n + nh];
  }
  for (int j = 0; j < ne; ++j) {
    for (int a = 0; a < qh; ++a) {
      BE[j * qe + a] = 0.5 * (T[a * n + j] + T[(q - 1 - a) * n + j]);
      BO[j * qh + a] = 0.5 * (T[a * n + j] - T[(q - 1 - a) * n + j]);
    }
    if (q & 1) BE[j * qe + qh] = T[qh * n + j];
  }
}

// 1D finite element interpolation from a coarse element to its two children (GMG prolongation,
// DESIGN.md reading R23): M[t][i] = l_i(xi_c(t)), t = 0 .. 2p indexes the 2p+1 fine GLL nodes of
// the two children, xi_c(t) = (s + xi_{t - s p}) / 2 with s = (t >= p); barycentric Lagrange on
// the coarse GLL nodes (exact at coincident nodes).  M has (2p+1) x (p+1) doubles.
int host_prolongation_1d(int p, double* M) {
  if (p < 1 || p > 8) return ELAS_EINVAL;
  const int n = p + 1;
  std::vector<double> xi(n), bw(n);
  gll_nodes(p, xi.data());
  for (int i = 0; i < n; ++i) {
    double prod = 1.0;
    for (int j = 0; j < n; ++j)
      if (j != i) prod *= (xi[i] - xi[j]);
    bw[i] = 1.0 / prod;
  }
  for (int t = 0; t <= 2 * p; ++t) {
    const int sidx = t >= p ? 1 : 0;
    const double xc = 0.5 * (sidx + xi[t - sidx * p]);
    int hit = -1;
    for (int k = 0; k < n; ++k)
      if (xc == xi[k]) hit = k;
    double denom = 0.0;
    if (hit < 0)
      for (int j = 0; j < n; ++j) denom += bw[j] / (xc - xi[j]);
    for (int i = 0; i < n; ++i)
      M[t * n + i] = hit >= 0 ? (i == hit ? 1.0 : 0.0) : (bw[i] / (xc - xi[i])) / denom;
  }
  return ELAS_OK;
}

}  // namespace elas
