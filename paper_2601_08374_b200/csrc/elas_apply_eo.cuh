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

// CTA size and register target of the folded kernel per degree (ELAS_EO_NT_P<p>,
// ELAS_EO_MINB_P<p> override; measured by tools/ab_libs.sh)
// measured (tools/ab_libs.sh, config 4): 256 threads at p = 5 (EB = 5: 245 of 256 stage-X lines
// busy) 26.0 -> 28.5 GDoF/s; 160/192/224/256 lose at p = 3, 4, 6, 7, 8
template <int P> struct NtEO { static constexpr int value = P == 5 ? 256 : ELAS_NT; };
template <int P> struct MinbEO { static constexpr int value = P == 2 ? 4 : P == 3 ? 3 : MinBlocks<P>::value; };
#ifdef ELAS_EO_NT_P2
template <> struct NtEO<2> { static constexpr int value = ELAS_EO_NT_P2; };
#endif
#ifdef ELAS_EO_NT_P3
template <> struct NtEO<3> { static constexpr int value = ELAS_EO_NT_P3; };
#endif
#ifdef ELAS_EO_NT_P4
template <> struct NtEO<4> { static constexpr int value = ELAS_EO_NT_P4; };
#endif
#ifdef ELAS_EO_NT_P5
template <> struct NtEO<5> { static constexpr int value = ELAS_EO_NT_P5; };
#endif
#ifdef ELAS_EO_NT_P6
template <> struct NtEO<6> { static constexpr int value = ELAS_EO_NT_P6; };
#endif
#ifdef ELAS_EO_NT_P7
template <> struct NtEO<7> { static constexpr int value = ELAS_EO_NT_P7; };
#endif
#ifdef ELAS_EO_NT_P8
template <> struct NtEO<8> { static constexpr int value = ELAS_EO_NT_P8; };
#endif
#ifdef ELAS_EO_MINB_P2
template <> struct MinbEO<2> { static constexpr int value = ELAS_EO_MINB_P2; };
#endif
#ifdef ELAS_EO_MINB_P3
template <> struct MinbEO<3> { static constexpr int value = ELAS_EO_MINB_P3; };
#endif
#ifdef ELAS_EO_MINB_P4
template <> struct MinbEO<4> { static constexpr int value = ELAS_EO_MINB_P4; };
#endif
#ifdef ELAS_EO_MINB_P5
template <> struct MinbEO<5> { static constexpr int value = ELAS_EO_MINB_P5; };
#endif
#ifdef ELAS_EO_MINB_P6
template <> struct MinbEO<6> { static constexpr int value = ELAS_EO_MINB_P6; };
#endif
#ifdef ELAS_EO_MINB_P7
template <> struct MinbEO<7> { static constexpr int value = ELAS_EO_MINB_P7; };
#endif
#ifdef ELAS_EO_MINB_P8
template <> struct MinbEO<8> { static constexpr int value = ELAS_EO_MINB_P8; };
#endif

// register target of the FP32 (mixed-precision) instances: half-size registers leave room for more
// CTAs per SM where one element per CTA would otherwise cap the warps (p >= 7)
// (measured, config 4: p7 23.9 -> 41.3 GDoF/s at 4 CTAs/SM, p8 31.6 -> 40.9 at 3, p5 (256 threads)
// 35.8 -> 46.4 at 2)
#ifndef ELAS_EO32_MINB_LO
#define ELAS_EO32_MINB_LO 0
#endif
template <int P> struct MinbEO32 {
  static constexpr int value = P == 7 ? 4 : P == 8 ? 3 : P == 5 ? 2 : P == 6 ? 4
                               : (ELAS_EO32_MINB_LO > 0 ? ELAS_EO32_MINB_LO : MinbEO<P>::value);
};
// CTA size per precision: the FP32 p = 6 instance runs one element per 64-thread CTA, 4 CTAs/SM
// (measured, config 4: 52.7 -> 53.4 GDoF/s; the FP64 instance loses, 33.6 -> 33.3)
// FP64 p = 7: 96-thread CTAs (81 x-lines: 84 % of the lanes busy in stage X instead of 63 %):
// 24.2 -> 24.5 GDoF/s (round 2)
template <int P, typename T> struct NtEOT {
  static constexpr int value = (sizeof(T) == 4 && P == 6) ? 64 : (sizeof(T) == 8 && P == 7) ? 96 : NtEO<P>::value;
};

// Persistent CTAs (measured, config 4): a win only where ONE CTA fills an SM (p = 5: 256 threads,
// 167 KB smem) and nothing else covers a CTA's start-up latency: 28.4 -> 30.1 GDoF/s; elsewhere
// the second resident CTA already does and the loop costs registers (p6 33.4 -> 32.3).
template <int P> struct PersistEO { static constexpr bool value = P == 5; };
// Stage-Z gather with 32-bit word offsets (3 nodes < 2^31 per rank, checked by elas_create) and the
// L2::256B prefetch hint on the loads; measured (config 4, GDoF/s): p4 27.4 -> 28.4, p5 30.1 ->
// 30.5, p7 23.8 -> 24.3, p8 30.4 -> 30.7, but p6 33.5 -> 32.6 (its 255-register budget spills).
// Measured and rejected: waiting on the qdata ring per PAIR of points (p6 33.5 -> 33.0, p7 -5 %).
#ifndef ELAS_EO_G32_MASK
#define ELAS_EO_G32_MASK 0x1BC   // degrees (bit p) with the 32-bit gather: 2, 3, 4, 5, 7, 8
#endif
template <int P> struct G32EO { static constexpr bool value = ((ELAS_EO_G32_MASK >> P) & 1) != 0; };

// Odd Y-buffer line stride (Cfg LNO, pick_LN) per degree (bit p); measured (config 4, GDoF/s):
// FP64 p7 25.0 -> 27.2, FP32 p7 49.0 -> 49.2; p5 30.5 -> 29.2 and p3 23.9 -> 23.7 lose (their
// x-line conflicts are 2-way, the new stage-Y conflict costs more).  Walking stages Y/Yt a3-fast
// to keep them conflict-free at the odd stride measured 27.0 at p7 (rejected).
#ifndef ELAS_EO_LNO_MASK
#define ELAS_EO_LNO_MASK (1 << 7)
#endif
template <int P> struct LnoEO { static constexpr int value = (ELAS_EO_LNO_MASK >> P) & 1; };

template <int P, int Q, typename T = double>
using CfgEO = Cfg<P, Q, 2 * Fold<P, Q>::TS, NtEOT<P, T>::value, (int)sizeof(T), 1, LnoEO<P>::value>;

// Quadrature-data ring (ELAS_QD_RING = R > 0): every stage-X thread owns one x-line (EB q^2 <=
// NT), so it streams ITS line's 9 values per point into its own shared-memory slots with
// cp.async (LDGSTS, no registers, no CTA barrier), R-1 points ahead of the pointwise stage; the
// first R-1 points are requested at CTA start and land during stages Z and Y.  Slots are
// [R][9][NT] so both the copies and the reads are contiguous across a warp.
// measured (tools/ab_libs.sh, config 4): an aliased ring of 4 points helps at p >= 6
// (p6 29.9 -> 30.7, p8 27.5 -> 28.8 GDoF/s); at p <= 5 the Z buffer holds at most 2 slots per
// thread and the one-point register prefetch is as good or better.  Round 2 (96-thread CTAs and the
// 32-bit gather at p7): the one-point register prefetch beats the ring for the FP64 p7 instance
// (24.5 -> 25.05), ties at p6 (33.62 / 33.68) and loses at p8 (30.39 -> 29.78) and for FP32 p7
// (48.4 -> 40.0).
#ifndef ELAS_QD_RING
#define ELAS_QD_RING (P >= 6 ? 4 : 0)
#endif
// whole-CTA TMA staging of qdata where two CTAs fit (elas_apply.cuh); off at p = 2, which
// runs faster at 4 CTAs/SM without it (12.5 -> 16 GDoF/s)
// measured: p = 3 without staging at 3 CTAs/SM 21.4 -> 22.2
template <int P> struct StageEO { static constexpr bool value = P != 2 && P != 3; };
template <int P, int Q, typename T = double>
struct RingEO {
  using C = CfgEO<P, Q, T>;
  static constexpr int WB = (int)sizeof(T);
  // the ring lives in the Z buffer, idle during stage X (first copies issued after the stage-Y
  // barrier); a dedicated ring costs occupancy and lost everywhere
  static constexpr bool ALIAS = true;
  static constexpr int RMAX = ALIAS ? (C::EB * C::ZE) / (9 * C::NT) : 16;
  static constexpr int WANT = (WB == 8 && P == 7) ? 0 : ELAS_QD_RING;
  static constexpr int R0 = WANT < RMAX ? WANT : RMAX;
  static constexpr int R = R0 >= 2 ? R0 : 0;
  static constexpr bool STAGE = C::STAGE_QD && R == 0 && StageEO<P>::value;  // whole-CTA TMA staging
  static constexpr int OFF = ALIAS ? C::TAB : (C::TAB + C::EB * (C::ZE + C::YE) + C::AL - 1) & ~(C::AL - 1);
  static constexpr size_t smem = (R > 0 && !ALIAS) ? (size_t)WB * (size_t)(OFF + R * 9 * C::NT)
                                 : STAGE ? C::smem : (size_t)WB * (size_t)(C::TAB + C::EB * (C::ZE + C::YE));
};

template <typename T>
__device__ __forceinline__ void cp_async_w(T* dst, const T* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"((int)sizeof(T)) : "memory");
}

// sigma~ = r tr(H) I + H + H^T with H = G A~ ; F = sigma~ A~^T (elas_apply.cuh pointwise, any T)
template <typename T>
__device__ __forceinline__ void pointwise_t(T (&g)[3][3], const T (&A)[9], T r) {
  T H[3][3];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int m = 0; m < 3; ++m) H[c][m] = fma(g[c][2], A[6 + m], fma(g[c][1], A[3 + m], g[c][0] * A[m]));
  const T s = r * (H[0][0] + H[1][1] + H[2][2]);
  T S[3][3];
  S[0][0] = fma(T(2), H[0][0], s);
  S[1][1] = fma(T(2), H[1][1], s);
  S[2][2] = fma(T(2), H[2][2], s);
  S[0][1] = S[1][0] = H[0][1] + H[1][0];
  S[0][2] = S[2][0] = H[0][2] + H[2][0];
  S[1][2] = S[2][1] = H[1][2] + H[2][1];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int d = 0; d < 3; ++d)
      g[c][d] = fma(S[c][2], A[3 * d + 2], fma(S[c][1], A[3 * d + 1], S[c][0] * A[3 * d]));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Deterministic (colored) mode: the elements of one launch all have the same parity (cx, cy, cz)
// per axis, so no two of them share a node: each node receives ONE contribution per launch and
// the (fire-and-forget) atomic add y + v is order-free; the 8 colors run in a fixed order =>
// bitwise reproducible y.  A plain read-modify-write would
// be equally deterministic but exposes the load latency (measured 2x slower).  Linear index l in the launch -> (ix, iy, iz) of the color's lattice ->
// element (2 ix + cx, 2 iy + cy, 2 (iz + iz0) + cz).  on = 0: l is the element id itself.
struct ColorMap {
  int on, cx, cy, cz, ncx, ncy, iz0;
};

template <bool COLORED>
__device__ __forceinline__ int64_t elem_coords(const ColorMap& cm, const Slab& s, int64_t l, int& ex, int& ey,
                                               int& ez) {
  const uint32_t l32 = (uint32_t)l;
  if constexpr (!COLORED) {
    const uint32_t nx = (uint32_t)s.nx, ny = (uint32_t)s.ny;
    const uint32_t exy = l32 / nx;
    ex = (int)(l32 - exy * nx);
    ez = (int)(exy / ny);
    ey = (int)(exy - (uint32_t)ez * ny);
    return l;
  }
  const uint32_t ncx = (uint32_t)cm.ncx, ncy = (uint32_t)cm.ncy;
  const uint32_t ixy = l32 / ncx, ix = l32 - ixy * ncx, iz = ixy / ncy, iy = ixy - iz * ncy;
  ex = 2 * (int)ix + cm.cx;
  ey = 2 * (int)iy + cm.cy;
  ez = 2 * ((int)iz + cm.iz0) + cm.cz;
  return ex + (int64_t)s.nx * (ey + (int64_t)s.ny * ez);
}

// u (n values per component) -> even (ne) / odd (nh) halves
template <int N, int NE, int NHX, typename T>
__device__ __forceinline__ void fold_in(const T (&u)[3][N], T (&up)[3][NE], T (&um)[3][NHX]) {
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

// OTF (geometry on the fly, FP64): no stored quadrature data; each stage-X thread rebuilds A~ at
// its points from the element's trilinear-map coefficients (QD_LAYOUT_OTF, staged in shared
// memory with the Gauss points and sqrt weights): along an x-line dx/dxi1 is constant and
// dx/dxi2, dx/dxi3 are linear in xi1, so J costs 6 FMAs per point, then the adjugate, det and
// one rsqrt: A~ = sqrt(mu) sqrt(w1 w2 w3) adj(J) / sqrt(det J)  (= sqrt(mu W) J^{-1}).
template <int P, int Q, typename T>
struct OtfSmem {
  using C = CfgEO<P, Q, T>;
  static constexpr int OFFG = (C::TAB + C::EB * (C::ZE + C::YE) + 1) & ~1;   // gq[Q] | sqw[Q] | geo[EB][GEO]
  static constexpr size_t smem = sizeof(T) * (size_t)(OFFG + 2 * Q + C::EB * GEO_WORDS);
};

// ANISO (general anisotropic material, Eq. 2): the stored qdata is
// A~ = sqrt(W) J^{-1} (mu = 1, r = 0 at setup) and every element carries its 6 x 6 Voigt matrix
// (21 upper-triangle words, staged per batch in shared memory).  At a point: H = G A~ =
// sqrt(W) grad u, eps_v = [H11, H22, H33, H23 + H32, H13 + H31, H12 + H21] (engineering shear,
// PAPER.md:162), sigma_v = C eps_v, F = sigma~ A~^T = W sigma J^{-T}.
constexpr int C21 = 21;
template <int P, int Q, typename T>
struct AnisoSmem {
  using C = CfgEO<P, Q, T>;
  using RG = RingEO<P, Q, T>;
  static constexpr int OFFC = RG::STAGE ? ((C::BASE + C::EB * C::QDE + 2 + 1) & ~1)
                                        : ((C::TAB + C::EB * (C::ZE + C::YE) + 1) & ~1);
  static constexpr size_t smem = sizeof(T) * (size_t)(OFFC + C::EB * C21);
};

// upper-triangle index of the symmetric 6 x 6 Voigt matrix, row-major: (a, b), a <= b
__host__ __device__ constexpr int c21_index(int a, int b) {
  return a <= b ? a * 6 - a * (a - 1) / 2 + (b - a) : b * 6 - b * (b - 1) / 2 + (a - b);
}

template <typename T>
__device__ __forceinline__ void pointwise_aniso(T (&g)[3][3], const T (&A)[9], const T* __restrict__ Cs) {
  T H[3][3];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int m = 0; m < 3; ++m) H[c][m] = fma(g[c][2], A[6 + m], fma(g[c][1], A[3 + m], g[c][0] * A[m]));
  const T ev[6] = {H[0][0], H[1][1], H[2][2], H[1][2] + H[2][1], H[0][2] + H[2][0], H[0][1] + H[1][0]};
  T sv[6];
#pragma unroll
  for (int a = 0; a < 6; ++a) {
    T acc = 0;
#pragma unroll
    for (int b = 0; b < 6; ++b) acc = fma(Cs[c21_index(a, b)], ev[b], acc);
    sv[a] = acc;
  }
  const T S[3][3] = {{sv[0], sv[5], sv[4]}, {sv[5], sv[1], sv[3]}, {sv[4], sv[3], sv[2]}};
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int d = 0; d < 3; ++d)
      g[c][d] = fma(S[c][2], A[3 * d + 2], fma(S[c][1], A[3 * d + 1], S[c][0] * A[3 * d]));
}

// Folded tables in the CONSTANT bank (ELAS_EO_CTAB): every coefficient index of the folded
// contractions is a compile-time constant after unrolling and warp-uniform, so ptxas fetches the
// coefficients with uniform-datapath LDCU (SASS `LDCU.128 URx, c[0x3][imm]`) instead of per-thread
// shared-memory loads, and the CTA prologue has no table copy.  The tables depend on (p, q) only (GLL nodes, Gauss points), so one
// copy per (P, Q, T) serves every operator; apply_eo_upload_p<P> writes it at elas_create.
// Per (degree, precision, geometry mode) a mask of the stages that read the constant bank:
// 1 = forward Z, Y; 2 = X; 4 = transposed Yt, Zt (7 = all; 5 = all but stage X, where the
// x-line's gradients hold most registers); the others read the shared-memory copy, which the
// prologue fills from the constant bank with bit 8 set, else from global memory.  Measured (config 4, GDoF/s, shared -> constant; FP64 /
// FP32 / geometry on the fly): p2 (all stages) 16.7 -> 18.6 / 23.5 -> 24.7 / 13.0 -> 15.4
// (anisotropic 12.3 -> 12.8);
// stages Z/Y only: p3 22.2 -> 23.3 / 32.7 -> 34.3 / 20.7 -> 21.7, p4 26.2 -> 26.9 / 42.4 -> 43.4
// / 22.9 -> 23.7, p5 30.1 -> 26.9 (lost) / 45.2 -> 45.9 / 26.0 -> 26.5, p6 33.4 -> 31.0 (lost) /
// 50.6 -> 52.8 / 33.1 -> 31.4 (lost), p7, p8 lost everywhere; all stages at p3..p8 FP64 lost
// 8-40 %; forward stages only (mask 1): FP64 p4 26.8 -> 27.2, p6 33.4 -> 31.7, config 5
// 33.5 -> 31.9; forward + X (mask 3): FP32 p4 43.5 -> 44.4.  Prologue fill from the constant
// bank (bit 8) on top: FP64 p3 23.3 -> 23.7 (13), p4 27.3 -> 27.6 (9), p6 33.4 -> 33.6, p7 23.3 ->
// 23.5, p8 29.4 -> 29.6 (8); on the fly p5 26.5 -> 27.1 (13); FP32 no gain.  Per-thread LDC into
// general registers (bit 16) for stage X (mask 26): FP32 p5 46.0 -> 47.8, FP64 p8 29.7 -> 30.1,
// on the fly p7 22.0 -> 22.3; every other degree loses 1-15 % (one LDC issued per coefficient use;
// all stages: p6 33.6 -> 31.9).  Where the constant bank loses, the coefficients hoisted into
// registers push the register-capped kernels into spills, and a DFMA with a uniform-register
// operand issues at about half rate.  ELAS_EO_CTAB = mask / -1 overrides.
#ifndef ELAS_EO_CTAB
#define ELAS_EO_CTAB 0
#endif
template <int P, typename T, bool OTF, bool ANISO>
struct CtabEO {
  static constexpr int tuned = P == 2 ? 7
                               : ANISO          ? 8   // p3 19.8 -> 17.4, p4 22.0 -> 21.8 (stages Z/Y)
                               : sizeof(T) == 4 ? (P == 4 ? 3 : P == 5 ? 26 : P >= 3 && P <= 6 ? 5 : 0)
                               : OTF            ? (P >= 3 && P <= 5 ? 13 : P == 7 ? 26 : 8)
                                                : (P == 3 ? 13 : P == 4 ? 9 : P == 8 ? 26 : 8);
  static constexpr int value = ELAS_EO_CTAB == 0 ? tuned : ELAS_EO_CTAB < 0 ? 0 : ELAS_EO_CTAB;
};
template <int P, int Q, typename T>
__constant__ T c_fold[2 * Fold<P, Q>::TS];

template <int P, int Q, typename T, bool COLORED, bool OTF = false, bool ANISO = false>
__global__ void __launch_bounds__(CfgEO<P, Q, T>::NT, sizeof(T) == 4 ? MinbEO32<P>::value : MinbEO<P>::value)
    apply_eo_kernel(const double* __restrict__ x, double* __restrict__ y, const T* __restrict__ qd,
                    const double* __restrict__ rr, const T* __restrict__ tables, Slab s,
                    int64_t e_begin, int64_t e_end, int pref_ctas, ColorMap cm,
                    const double* __restrict__ cc) {
  using C = CfgEO<P, Q, T>;
  using F = Fold<P, Q>;
  constexpr int N = C::N, NT = C::NT, EB = C::EB;
  constexpr int NE = F::NE, NH = F::NH, QE = F::QE, QH = F::QH, NHX = F::NHX;
  using RG = RingEO<P, Q, T>;
  constexpr int R = OTF ? 0 : RG::R;
  constexpr bool STG = RG::STAGE && !OTF;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  constexpr int CTM = CtabEO<P, T, OTF, ANISO>::value;   // constant-bank stages (mask, above)
  constexpr bool CT = (CTM & 7) == 7;                     // no stage reads the shared copy
  // bit 16: per-thread LDC into general registers (the offset is zero at run time but not provably
  // warp-uniform, so ptxas cannot route the coefficient through a uniform register: DFMA keeps
  // all-register operands, and the coefficients stay off the shared-memory pipe)
  const int cz = (CTM & 16) ? (int)threadIdx.x * (int)(gridDim.z - 1) : 0;
  const T* tB = (CTM & 1) ? c_fold<P, Q, T> + cz : smem;  // stages Z, Y: folded B (parity +1)
  const T* tD = (CTM & 1) ? c_fold<P, Q, T> + F::TS + cz : smem + F::TS;  // folded D (parity -1)
  const T* xB = (CTM & 2) ? c_fold<P, Q, T> + cz : smem;  // stage X
  const T* xD = (CTM & 2) ? c_fold<P, Q, T> + F::TS + cz : smem + F::TS;
  const T* bB = (CTM & 4) ? c_fold<P, Q, T> + cz : smem;  // stages Yt, Zt
  const T* bD = (CTM & 4) ? c_fold<P, Q, T> + F::TS + cz : smem + F::TS;
  T* sZ = smem + C::TAB;
  T* sY = sZ + EB * C::ZE;
  T* sQ = smem + C::BASE;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + C::BASE + EB * C::QDE);

  const int tid = threadIdx.x;
  // PST (persistent CTAs, p = 5): the grid covers the resident CTAs and each walks the
  // batches b, b + gridDim.x, ...; the next batch's z-columns are gathered into registers right
  // after the stage-Yt barrier so the loads fly during stage Zt, and the tables load once.
  constexpr bool PST = PersistEO<P>::value && !COLORED && !OTF && !ANISO;
  static_assert(EB * N * N <= NT, "stage Z assumes at most one z-column per thread");
  const int64_t plane = (int64_t)s.Nx * s.Ny;
  const bool bc = s.faces != 0;
  const int zi = tid % N, zj = (tid / N) % N, zel = tid / (N * N);
  const int64_t nbatch = (e_end - e_begin + EB - 1) / EB;
  const int64_t bstride = PST ? (int64_t)gridDim.x : nbatch;
  // Stage-Z gather issued before the table copy and the first barrier so that both global
  // latencies overlap (EB n^2 <= NT: at most one z-column per thread).  Element coordinates in
  // 32-bit arithmetic (element ids < 2^31).
  T u[3][N];
  auto gather = [&](int64_t batch) {
    const int64_t g0 = e_begin + batch * EB;
    const int gne = (int)((e_end - g0) < EB ? (e_end - g0) : EB);
    if (tid < gne * N * N) {
      int ex, ey, ez;
      elem_coords<COLORED>(cm, s, g0 + zel, ex, ey, ez);
      const int I = ex * P + zi, J = ey * P + zj;
      if constexpr (G32EO<P>::value) {
      // 32-bit word offsets; loads carry the L2::256B prefetch hint
      const uint32_t nodes32 = (uint32_t)s.nodes, plane32 = (uint32_t)plane;
      const double* xb = x + ((uint32_t)I + (uint32_t)s.Nx * (uint32_t)J + plane32 * (uint32_t)(ez * P));
#pragma unroll
      for (int k = 0; k < N; ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          ELAS_DCHECK((int64_t)(xb - x) + c * nodes32 + k * plane32 < 3 * s.nodes && xb >= x);
          double v;
          asm("ld.global.nc.L2::256B.f64 %0, [%1];" : "=d"(v) : "l"(xb + (c * nodes32 + k * plane32)));
          u[c][k] = (T)v;
        }
      if (bc) {
#pragma unroll
        for (int k = 0; k < N; ++k)
          if (is_constrained(I, J, ez * P + k, s)) {
#pragma unroll
            for (int c = 0; c < 3; ++c) u[c][k] = T(0);
          }
      }
      } else {
      const int64_t base = I + (int64_t)s.Nx * J + plane * ((int64_t)ez * P);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const bool cons = bc && is_constrained(I, J, ez * P + k, s);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          ELAS_DCHECK(base >= 0 && c * s.nodes + base + k * plane < 3 * s.nodes);
          u[c][k] = cons ? T(0) : (T)__ldg(x + c * s.nodes + base + k * plane);
        }
      }
      }
    }
  };
  gather(blockIdx.x);
  if constexpr (!CT && (CTM & 8)) {
    // the shared copy filled from the constant bank: LDC does not queue behind the gather's
    // DRAM misses in L1TEX the way the global table loads do
    for (int t = tid; t < 2 * F::TS; t += NT) smem[t] = c_fold<P, Q, T>[t];
  } else if constexpr (!CT) {
    const T* ft = tables + 2 * Q * N;   // fold(B) | fold(D) follow the plain tables
    for (int t = tid; t < 2 * F::TS; t += NT) smem[t] = ft[t];
  }
  if constexpr (STG) {
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  uint32_t phase = 0;

  for (int64_t batch = blockIdx.x; batch < nbatch; batch += bstride, phase ^= 1u) {
  const int64_t e0 = e_begin + batch * EB;
  const int ne = (int)((e_end - e0) < EB ? (e_end - e0) : EB);
  if constexpr (PST) __syncthreads();   // the previous batch is done with the Z tile and sQ
  if constexpr (STG) {
    if (tid == 0) {
      const uint32_t bar = smem_u32(mbar);
      const uint32_t bytes = (uint32_t)(sizeof(T) * ne * C::QDE);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
      if constexpr (!COLORED) {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sQ)),
            "l"(qd + e0 * (int64_t)C::QDE), "r"(bytes), "r"(bar)
            : "memory");
      } else {   // colored mode: the batch's elements are not contiguous, one bulk copy each
        for (int el = 0; el < ne; ++el) {
          int ex, ey, ez;
          const int64_t e = elem_coords<COLORED>(cm, s, e0 + el, ex, ey, ez);
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(sQ + el * C::QDE)),
              "l"(qd + e * (int64_t)C::QDE), "r"((uint32_t)(sizeof(T) * C::QDE)), "r"(bar)
              : "memory");
        }
      }
    }
  }
  // this thread's stage-X line (at most one: EB q^2 <= NT) and its qdata ring
  T* ring = smem + RG::OFF + tid;
  const bool has_line = tid < ne * Q * Q;
  int qex, qey, qez;
  const T* qline = qd + elem_coords<COLORED>(cm, s, e0 + tid / (Q * Q), qex, qey, qez) * (int64_t)C::QDE + tid % (Q * Q);
  auto ring_issue = [&](int a1) {
    if (has_line) {
#pragma unroll
      for (int f = 0; f < 9; ++f) cp_async_w(ring + ((a1 % (R > 0 ? R : 1)) * 9 + f) * NT, qline + (a1 * 9 + f) * Q * Q);
    }
    cp_async_commit();
  };
  if constexpr (R > 0 && !RG::ALIAS) {
#pragma unroll
    for (int a1 = 0; a1 < R - 1; ++a1) ring_issue(a1);
  }
  if constexpr (ANISO) {   // the batch's Voigt matrices
    T* cs = smem + AnisoSmem<P, Q, T>::OFFC;
    for (int t = tid; t < ne * C21; t += NT) {
      int cex, cey, cez;
      cs[t] = (T)cc[elem_coords<COLORED>(cm, s, e0 + t / C21, cex, cey, cez) * C21 + t % C21];
    }
  }
  if constexpr (OTF) {   // Gauss points, sqrt weights and the batch's Jacobian coefficients
    T* gs = smem + OtfSmem<P, Q, T>::OFFG;
    for (int t = tid; t < 2 * Q; t += NT) gs[t] = tables[2 * Q * N + 2 * F::TS + t];
    for (int t = tid; t < ne * GEO_WORDS; t += NT) {
      int gex, gey, gez;
      const int64_t ge = elem_coords<COLORED>(cm, s, e0 + t / GEO_WORDS, gex, gey, gez);
      const int w = t % GEO_WORDS;
      // p = 1 ops store the geometry lane-interleaved for the thread-per-element kernel (OTF32)
      gs[2 * Q + t] = P == 1 ? qd[(ge >> 5) * (int64_t)(32 * GEO_WORDS) + w * 32 + (ge & 31)]
                             : qd[ge * GEO_WORDS + w];
    }
  }
#if ELAS_L2_PREFETCH
  if (tid == 0 && pref_ctas > 0) {
    const int64_t pe0 = e0 + (int64_t)(PST ? (int)gridDim.x : pref_ctas) * EB;
    if (pe0 < e_end && !COLORED && !OTF) {   // (OTF: no quadrature data to prefetch)
      const int64_t pne = (e_end - pe0) < EB ? (e_end - pe0) : EB;
      const uintptr_t a0 = (uintptr_t)(qd + pe0 * (int64_t)C::QDE);
      const uintptr_t a1 = a0 + (uintptr_t)(pne * C::QDE * sizeof(T));
      const uintptr_t lo = a0 & ~(uintptr_t)15, hi = (a1 + 15) & ~(uintptr_t)15;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((uint32_t)(hi - lo)) : "memory");
    }
  }
#endif
  const bool zcol = tid < ne * N * N;
  __syncthreads();

  // ---------------- Stage Z: folded contraction in z of the gathered column -------------
  if (zcol) {
    const int i = zi, j = zj, el = zel;
    T up[3][NE], um[3][NHX];
    fold_in<N, NE, NHX>(u, up, um);
    T* dst = sZ + el * C::ZE + j * N + i;
#pragma unroll
    for (int a = 0; a < QE; ++a) {
      const bool mid = (Q & 1) && a == QH;
      T eb[3] = {0, 0, 0}, ob[3] = {0, 0, 0}, ed[3] = {0, 0, 0}, od[3] = {0, 0, 0};
#pragma unroll
      for (int k = 0; k < NE; ++k) {
        const T b = tB[F::FE + a * NE + k];
#pragma unroll
        for (int c = 0; c < 3; ++c) eb[c] = fma(b, up[c][k], eb[c]);
        if (!mid) {
          const T d = tD[F::FE + a * NE + k];
#pragma unroll
          for (int c = 0; c < 3; ++c) ed[c] = fma(d, up[c][k], ed[c]);
        }
      }
#pragma unroll
      for (int k = 0; k < NH; ++k) {
        const T d = tD[F::FO + a * NH + k];
#pragma unroll
        for (int c = 0; c < 3; ++c) od[c] = fma(d, um[c][k], od[c]);
        if (!mid) {
          const T b = tB[F::FO + a * NH + k];
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
    const T* src = sZ + el * C::ZE + a3 * C::SA + i;
    T bp[3][NE], bm[3][NHX], dp[3][NE], dm[3][NHX];
    {
      T zb[3][N], zd[3][N];
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
    T* dst = sY + el * C::YE + a3 * C::LN + i;
#pragma unroll
    for (int a2 = 0; a2 < QE; ++a2) {
      const bool mid = (Q & 1) && a2 == QH;
      // y0 = By zb (+1), y1 = Dy zb (-1), y2 = By zd (+1)
      T e0[3] = {0, 0, 0}, o0[3] = {0, 0, 0}, e1[3] = {0, 0, 0}, o1[3] = {0, 0, 0};
      T e2[3] = {0, 0, 0}, o2[3] = {0, 0, 0};
#pragma unroll
      for (int j = 0; j < NE; ++j) {
        const T b = tB[F::FE + a2 * NE + j];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          e0[c] = fma(b, bp[c][j], e0[c]);
          e2[c] = fma(b, dp[c][j], e2[c]);
        }
        if (!mid) {
          const T d = tD[F::FE + a2 * NE + j];
#pragma unroll
          for (int c = 0; c < 3; ++c) e1[c] = fma(d, bp[c][j], e1[c]);
        }
      }
#pragma unroll
      for (int j = 0; j < NH; ++j) {
        const T d = tD[F::FO + a2 * NH + j];
#pragma unroll
        for (int c = 0; c < 3; ++c) o1[c] = fma(d, bm[c][j], o1[c]);
        if (!mid) {
          const T b = tB[F::FO + a2 * NH + j];
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
  if constexpr (R > 0 && RG::ALIAS) {   // the Z buffer is free now
#pragma unroll
    for (int a1 = 0; a1 < R - 1; ++a1) ring_issue(a1);
  }
  if constexpr (STG) {
    const uint32_t bar = smem_u32(mbar);
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(bar), "r"(phase)
        : "memory");
  }
  for (int w = tid; w < ne * Q * Q; w += NT) {
    const int L = w % (Q * Q), el = w / (Q * Q);
    const int a3 = L % Q, a2 = L / Q;
    int xex, xey, xez;
    const int64_t e = elem_coords<COLORED>(cm, s, e0 + el, xex, xey, xez);
    T* line = sY + el * C::YE + a2 * C::S2 + a3 * C::LN;
    T g[3][3][Q];
#pragma unroll
    for (int v = 0; v < 3; ++v) {
      const T* tab = (v == 0) ? xD : xB;   // x-derivative for v = 0 (parity -1)
      const bool odd = (v == 0);
      T fp[3][NE], fm[3][NHX];
      {
        T f[3][N];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int i = 0; i < N; ++i) f[c][i] = line[c * C::YC + v * C::YV + i];
        fold_in<N, NE, NHX>(f, fp, fm);
      }
#pragma unroll
      for (int a1 = 0; a1 < QE; ++a1) {
        const bool mid = (Q & 1) && a1 == QH;
        T ev[3] = {0, 0, 0}, ov[3] = {0, 0, 0};
        if (!(mid && odd)) {
#pragma unroll
          for (int i = 0; i < NE; ++i) {
            const T t = tab[F::FE + a1 * NE + i];
#pragma unroll
            for (int c = 0; c < 3; ++c) ev[c] = fma(t, fp[c][i], ev[c]);
          }
        }
        if (!(mid && !odd)) {
#pragma unroll
          for (int i = 0; i < NH; ++i) {
            const T t = tab[F::FO + a1 * NH + i];
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
    ELAS_DCHECK(e >= 0 && e < (int64_t)s.nx * s.ny * s.nz && xex < s.nx && xey < s.ny && xez < s.nz);
    const T r = (T)__ldg(rr + e);
    const T* qp = STG ? sQ + el * C::QDE + L : qd + e * (int64_t)C::QDE + L;
    // geometry on the fly: per-line constants
    T col1[3], b2[3], s2[3], b3[3], s3[3], sq = 0;
    const T* gs = smem + OtfSmem<P, Q, T>::OFFG;
    if constexpr (OTF) {
      const T* ge = gs + 2 * Q + el * GEO_WORDS;
      const T xi2 = gs[a2], xi3 = gs[a3];
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        col1[m] = fma(fma(ge[9 + m], xi3, ge[3 + m]), xi2, fma(ge[6 + m], xi3, ge[m]));
        b2[m] = fma(ge[18 + m], xi3, ge[12 + m]);
        s2[m] = fma(ge[21 + m], xi3, ge[15 + m]);
        b3[m] = fma(ge[30 + m], xi2, ge[24 + m]);
        s3[m] = fma(ge[33 + m], xi2, ge[27 + m]);
      }
      sq = ge[36] * gs[Q + a2] * gs[Q + a3];
    }
    T An[9];
    if constexpr (R == 0 && !OTF) {
#pragma unroll
      for (int f = 0; f < 9; ++f) An[f] = qp[f * Q * Q];
    }
#pragma unroll
    for (int a1 = 0; a1 < Q; ++a1) {
      T A[9];
      if constexpr (OTF) {
        const T xi1 = gs[a1];
        T J[3][3];
#pragma unroll
        for (int m = 0; m < 3; ++m) {
          J[m][0] = col1[m];
          J[m][1] = fma(s2[m], xi1, b2[m]);
          J[m][2] = fma(s3[m], xi1, b3[m]);
        }
        T adj[3][3];
        adj[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
        adj[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
        adj[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
        adj[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
        adj[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
        adj[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
        adj[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
        adj[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
        adj[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        const T det = J[0][0] * adj[0][0] + J[0][1] * adj[1][0] + J[0][2] * adj[2][0];
        const T sc = sq * gs[Q + a1] * rsqrt(det);
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int m = 0; m < 3; ++m) A[3 * d + m] = sc * adj[d][m];
      } else if constexpr (R > 0) {
        if (a1 + R - 1 < Q) ring_issue(a1 + R - 1);
        else cp_async_commit();                    // empty group keeps the count uniform
        cp_async_wait<R - 1>();                    // this thread's copies of point a1 landed
#pragma unroll
        for (int f = 0; f < 9; ++f) A[f] = ring[((a1 % R) * 9 + f) * NT];
      } else {
#pragma unroll
        for (int f = 0; f < 9; ++f) A[f] = An[f];
        if (a1 + 1 < Q) {
#pragma unroll
          for (int f = 0; f < 9; ++f) An[f] = qp[((a1 + 1) * 9 + f) * Q * Q];
        }
      }
      T G[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) G[c][d] = g[c][d][a1];
      if constexpr (ANISO) pointwise_aniso<T>(G, A, smem + AnisoSmem<P, Q, T>::OFFC + el * C21);
      else pointwise_t<T>(G, A, r);
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) g[c][d][a1] = G[c][d];
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const T* tab = (d == 0) ? xD : xB;
      const bool odd = (d == 0);
      // fold over the points a1 in place: g[.][a] <- g_a + g_{q-1-a}, g[.][q-1-a] <- g_a - g_{q-1-a}
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int a = 0; a < QH; ++a) {
          const T lo = g[c][d][a], hi = g[c][d][Q - 1 - a];
          g[c][d][a] = lo + hi;
          g[c][d][Q - 1 - a] = lo - hi;
        }
#pragma unroll
      for (int i = 0; i < NE; ++i) {
        const bool mid = (N & 1) && i == NH;
        T ev[3] = {0, 0, 0}, ov[3] = {0, 0, 0};
        if (!(mid && odd)) {
#pragma unroll
          for (int a = 0; a < QE; ++a) {
            const T t = tab[F::BE + i * QE + a];
#pragma unroll
            for (int c = 0; c < 3; ++c) ev[c] = fma(t, g[c][d][a], ev[c]);
          }
        }
        if (!(mid && !odd)) {
#pragma unroll
          for (int a = 0; a < QH; ++a) {
            const T t = tab[F::BO + i * QH + a];
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
    const T* src = sY + el * C::YE + a3 * C::LN + i;
    // wb = By^T V0 + Dy^T V1, wd = By^T V2 ; X/Y sums per node pair (j, n-1-j)
    T bX[3][NE], bY[3][NE], dX[3][NE], dY[3][NE];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < NE; ++j) bX[c][j] = bY[c][j] = dX[c][j] = dY[c][j] = 0.0;
#pragma unroll
    for (int a = 0; a < QE; ++a) {
      const bool mid = (Q & 1) && a == QH;
      T v0p[3], v0m[3], v1p[3], v1m[3], v2p[3], v2m[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const T l0 = src[c * C::YC + a * C::S2];
        const T l1 = src[c * C::YC + C::YV + a * C::S2];
        const T l2 = src[c * C::YC + 2 * C::YV + a * C::S2];
        if (mid) {
          v0p[c] = l0; v1p[c] = l1; v2p[c] = l2;
          v0m[c] = v1m[c] = v2m[c] = 0.0;
        } else {
          const T h0 = src[c * C::YC + (Q - 1 - a) * C::S2];
          const T h1 = src[c * C::YC + C::YV + (Q - 1 - a) * C::S2];
          const T h2 = src[c * C::YC + 2 * C::YV + (Q - 1 - a) * C::S2];
          v0p[c] = l0 + h0; v0m[c] = l0 - h0;
          v1p[c] = l1 + h1; v1m[c] = l1 - h1;
          v2p[c] = l2 + h2; v2m[c] = l2 - h2;
        }
      }
#pragma unroll
      for (int j = 0; j < NE; ++j) {
        const bool jmid = (N & 1) && j == NH;
        const T be = bB[F::BE + j * QE + a];
        const T de = bD[F::BE + j * QE + a];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          bX[c][j] = fma(be, v0p[c], bX[c][j]);
          dX[c][j] = fma(be, v2p[c], dX[c][j]);
          if (!jmid) bY[c][j] = fma(de, v1p[c], bY[c][j]);
        }
        if (!mid) {
          const T bo = bB[F::BO + j * QH + a];
          const T dO = bD[F::BO + j * QH + a];
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
    T* dst = sZ + el * C::ZE + a3 * C::SA + i;
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
  if constexpr (PST) {
    if (batch + bstride < nbatch) gather(batch + bstride);   // in flight during stage Zt
  }

  // ---------------- Stage Zt: folded transposed contraction in z + scatter-add ----------
  for (int w = tid; w < ne * N * N; w += NT) {
    const int i = w % N, j = (w / N) % N, el = w / (N * N);
    int ex, ey, ez;
    elem_coords<COLORED>(cm, s, e0 + el, ex, ey, ez);
    const T* src = sZ + el * C::ZE + j * N + i;
    T X[3][NE], Y[3][NE];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int k = 0; k < NE; ++k) X[c][k] = Y[c][k] = 0.0;
#pragma unroll
    for (int a = 0; a < QE; ++a) {
      const bool mid = (Q & 1) && a == QH;
      T wbp[3], wbm[3], wdp[3], wdm[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const T lb = src[c * C::ZC + a * C::SA], ld = src[c * C::ZC + C::ZV + a * C::SA];
        if (mid) {
          wbp[c] = lb; wdp[c] = ld; wbm[c] = wdm[c] = 0.0;
        } else {
          const T hb = src[c * C::ZC + (Q - 1 - a) * C::SA];
          const T hd = src[c * C::ZC + C::ZV + (Q - 1 - a) * C::SA];
          wbp[c] = lb + hb; wbm[c] = lb - hb;
          wdp[c] = ld + hd; wdm[c] = ld - hd;
        }
      }
#pragma unroll
      for (int k = 0; k < NE; ++k) {
        const bool kmid = (N & 1) && k == NH;
        const T be = bB[F::BE + k * QE + a];
        const T de = bD[F::BE + k * QE + a];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          X[c][k] = fma(be, wbp[c], X[c][k]);
          if (!kmid) Y[c][k] = fma(de, wdp[c], Y[c][k]);
        }
        if (!mid) {
          const T bo = bB[F::BO + k * QH + a];
          const T dO = bD[F::BO + k * QH + a];
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
    ELAS_DCHECK(base >= 0 && 2 * s.nodes + base + (N - 1) * plane < 3 * s.nodes && I < s.Nx && J < s.Ny);
#pragma unroll
    for (int k = 0; k < NE; ++k) {
      const bool kmid = (N & 1) && k == NH;
      if (!(bc && is_constrained(I, J, ez * P + k, s))) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double* dst = y + c * s.nodes + base + k * plane;
          const double v = (double)(kmid ? X[c][k] : X[c][k] + Y[c][k]);
          atomicAdd(dst, v);   // colored mode: one contribution per node per launch => order-free
        }
      }
      if (!kmid && !(bc && is_constrained(I, J, ez * P + N - 1 - k, s))) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double* dst = y + c * s.nodes + base + (N - 1 - k) * plane;
          const double v = (double)(X[c][k] - Y[c][k]);
          atomicAdd(dst, v);
        }
      }
    }
  }
  }   // batch loop
}

template <int P, int Q, typename T, bool COLORED, bool OTF = false, bool ANISO = false>
cudaError_t launch_apply_eo_pqc(const Slab& s, const double* x, double* y, const void* qd, const double* rr,
                                const void* tables, int64_t e_begin, int64_t e_end, cudaStream_t st,
                                const ColorMap& cm, const double* cc = nullptr) {
  using C = CfgEO<P, Q, T>;
  constexpr size_t SMEM = OTF ? OtfSmem<P, Q, T>::smem : ANISO ? AnisoSmem<P, Q, T>::smem : RingEO<P, Q, T>::smem;
  static KernelPrep prep;   // per device: the shared-memory attribute and the resident-CTA count
  int pref = 0;
  cudaError_t err = prep.prep(apply_eo_kernel<P, Q, T, COLORED, OTF, ANISO>, C::NT, SMEM, &pref);
  if (err != cudaSuccess) return err;
  const int64_t ne = e_end - e_begin;
  if (ne <= 0) return cudaSuccess;
  const int64_t nb = (ne + C::EB - 1) / C::EB;
  constexpr bool PST = PersistEO<P>::value && !COLORED && !OTF && !ANISO;
  const int64_t grid = PST ? (nb < pref ? nb : pref) : nb;
  apply_eo_kernel<P, Q, T, COLORED, OTF, ANISO><<<(unsigned)grid, C::NT, SMEM, st>>>(
      x, y, static_cast<const T*>(qd), rr, static_cast<const T*>(tables), s, e_begin, e_end, pref, cm, cc);
  return cudaGetLastError();
}

// fine-grained FP64 kernel (elas_apply_fg.cuh), per-degree mask (bit p).  Measured (config 4,
// GDoF/s, x-line -> FG): p6 33.46 -> 39.36, p7 26.89 -> 34.31, p8 30.29 -> 32.41, config 5 33.55 ->
// 37.51, p5 30.48 -> 30.87 (warp-padded X items, 4 CTAs/SM); p3 23.90 -> 16.86, p4 28.42 -> 25.63
// stay on the x-line kernel.
#ifndef ELAS_FG_MASK
#define ELAS_FG_MASK 0x1E0
#endif
template <int P> struct FgOn { static constexpr bool value = ((ELAS_FG_MASK >> P) & 1) != 0; };
#ifndef ELAS_FG_COLORED
#define ELAS_FG_COLORED 1   // deterministic (colored) mode on the fine-grained kernel too (config 4 p6: 27.1 -> 36.1 GDoF/s)
#endif
template <int P> struct FgColored { static constexpr bool value = ELAS_FG_COLORED != 0; };
#ifndef ELAS_FG_OTF
#define ELAS_FG_OTF 1   // geometry on the fly on the fine-grained kernel too (config 4 GDoF/s x-line -> FG:
                        // p5 27.7 -> 28.1, p6 33.6 -> 34.8, p7 24.3 -> 32.2, p8 30.0 -> 33.1; config 5 33.7 -> 34.8)
#endif
template <int P> struct FgOtf { static constexpr bool value = ELAS_FG_OTF != 0; };
#ifndef ELAS_FG_ANISO
#define ELAS_FG_ANISO 1   // anisotropic material (Eq. 2) on the fine-grained kernel too (config 4 GDoF/s
                          // x-line -> FG: p5 26.0 -> 29.0, p6 31.3 -> 36.1, p7 23.8 -> 32.4, p8 27.3 -> 32.2)
#endif
template <int P> struct FgAniso { static constexpr bool value = ELAS_FG_ANISO != 0; };
template <int P, int Q>
cudaError_t launch_apply_fg(const Slab& s, const double* x, double* y, const void* qd, const double* rr,
                            int64_t e_begin, int64_t e_end, cudaStream_t st, const ColorMap& cm, int otf,
                            const double* tables, const double* cc);
template <int P, int Q> void info_fg_pq(ApplyLaunch* info);

template <int P, int Q, typename T>
cudaError_t launch_apply_eo_pq(const Slab& s, const double* x, double* y, const void* qd, const double* rr,
                               const void* tables, int64_t e_begin, int64_t e_end, cudaStream_t st,
                               const ColorMap& cm, int otf, const double* cc) {
  if constexpr (sizeof(T) == 8 && FgOn<P>::value) {
    if ((!cc || FgAniso<P>::value) && (!cm.on || FgColored<P>::value) && (!otf || FgOtf<P>::value))
      return launch_apply_fg<P, Q>(s, x, y, qd, rr, e_begin, e_end, st, cm, otf, static_cast<const double*>(tables), cc);
  }
  if constexpr (sizeof(T) == 8) {
    if (cc)
      return cm.on ? launch_apply_eo_pqc<P, Q, T, true, false, true>(s, x, y, qd, rr, tables, e_begin, e_end, st, cm, cc)
                   : launch_apply_eo_pqc<P, Q, T, false, false, true>(s, x, y, qd, rr, tables, e_begin, e_end, st, cm, cc);
    if (otf)
      return cm.on ? launch_apply_eo_pqc<P, Q, T, true, true>(s, x, y, qd, rr, tables, e_begin, e_end, st, cm)
                   : launch_apply_eo_pqc<P, Q, T, false, true>(s, x, y, qd, rr, tables, e_begin, e_end, st, cm);
  }
  return cm.on ? launch_apply_eo_pqc<P, Q, T, true>(s, x, y, qd, rr, tables, e_begin, e_end, st, cm)
               : launch_apply_eo_pqc<P, Q, T, false>(s, x, y, qd, rr, tables, e_begin, e_end, st, cm);
}

template <int P, int Q, typename T>
void info_eo_pq(ApplyLaunch* info) {
  if constexpr (sizeof(T) == 8 && FgOn<P>::value) {
    info_fg_pq<P, Q>(info);
    return;
  }
  using C = CfgEO<P, Q, T>;
  info->threads = C::NT;
  info->elems_per_cta = C::EB;
  info->smem_bytes = RingEO<P, Q, T>::smem;
}

}  // namespace elas

// write the folded tables (host, 2 * TS doubles: fold(B) | fold(D)) into the constant bank of
// the FP64 and FP32 instances
namespace elas {
template <int P, int Q>
cudaError_t upload_eo_pq(const double* fold) {
  constexpr int n = 2 * Fold<P, Q>::TS;
  float f[n];
  for (int i = 0; i < n; ++i) f[i] = (float)fold[i];
  cudaError_t e = cudaMemcpyToSymbol(c_fold<P, Q, double>, fold, sizeof(double) * n);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_fold<P, Q, float>, f, sizeof(float) * n);
  return e;
}
}  // namespace elas

#define ELAS_DEFINE_DEGREE_EO(P)                                                                \
  ELAS_DCHECK_READER(dcheck_eo_p##P)                                                            \
  namespace elas {                                                                              \
  cudaError_t apply_eo_info_p##P(int q, int fp32, ApplyLaunch* info) {                          \
    if (q == P + 1) fp32 ? info_eo_pq<P, P + 1, float>(info) : info_eo_pq<P, P + 1, double>(info); \
    else if (q == P + 2) fp32 ? info_eo_pq<P, P + 2, float>(info) : info_eo_pq<P, P + 2, double>(info); \
    else return cudaErrorInvalidValue;                                                          \
    return cudaSuccess;                                                                         \
  }                                                                                             \
  cudaError_t apply_eo_upload_p##P(int q, const double* fold) {                                 \
    if (q == P + 1) return upload_eo_pq<P, P + 1>(fold);                                        \
    if (q == P + 2) return upload_eo_pq<P, P + 2>(fold);                                        \
    return cudaSuccess;                                                                         \
  }                                                                                             \
  cudaError_t apply_eo_launch_p##P(int q, int fp32, const Slab& s, const double* x, double* y,  \
                                   const void* qd, const double* rr, const void* tables,        \
                                   int64_t e_begin, int64_t e_end, cudaStream_t st,             \
                                   const int* color, int otf, const double* cc) {               \
    ColorMap cm{0, 0, 0, 0, 0, 0, 0};                                                           \
    if (color) cm = ColorMap{1, color[0], color[1], color[2], color[3], color[4], color[5]};    \
    if (q == P + 1)                                                                             \
      return fp32 ? launch_apply_eo_pq<P, P + 1, float>(s, x, y, qd, rr, tables, e_begin, e_end, st, cm, 0, nullptr) \
                  : launch_apply_eo_pq<P, P + 1, double>(s, x, y, qd, rr, tables, e_begin, e_end, st, cm, otf, cc); \
    if (q == P + 2)                                                                             \
      return fp32 ? launch_apply_eo_pq<P, P + 2, float>(s, x, y, qd, rr, tables, e_begin, e_end, st, cm, 0, nullptr) \
                  : launch_apply_eo_pq<P, P + 2, double>(s, x, y, qd, rr, tables, e_begin, e_end, st, cm, otf, cc); \
    return cudaErrorInvalidValue;                                                               \
  }                                                                                             \
  }
