// The operator object behind the opaque elas_op handle (shared by elas_api.cu and
// elas_solver.cu; not part of the public ABI).
#pragma once
#include <nccl.h>

#include <vector>

#include "elas_internal.h"

struct elas_op {
  int p = 0, q = 0, rank = 0, nranks = 1;
  int variant = ELAS_VARIANT_SIMT;  // resolved kernel variant
  bool deterministic = false;       // colored scatter (elas_set_deterministic)
  int32_t ez0 = 0, ez1 = 0;
  int32_t nz_global = 0;              // element layers of the whole mesh (all slabs)
  elas::Slab slab{};
  int device = 0;
  bool external = false;            // nranks > 1 without a communicator
  double* qd = nullptr;             // 9 q^3 doubles per element
  double* rr = nullptr;             // lambda/mu per element
  double* cc = nullptr;             // anisotropic ops: 21 Voigt words per element (elas_create_aniso)
  double* tab = nullptr;            // B | D | fold(B) | fold(D)
  float* tabf = nullptr;            // FP32 copy of tab (mixed-precision folded kernel)
  double* xs = nullptr;             // staging for elas_apply_host
  double* ys = nullptr;
  cudaStream_t h2d = nullptr, d2h = nullptr;   // copy streams of the chunked host apply
  std::vector<cudaEvent_t> host_ev;            // per chunk: x landed, chunk computed
  double *abl_E = nullptr, *abl_Eo = nullptr, *abl_Q = nullptr, *abl_G = nullptr;   // ablation-stage scratch
  cudaStream_t stream = nullptr;
  // multi-GPU
  ncclComm_t comm = nullptr;
  bool comm_borrowed = false;        // a coarser GMG level sharing the finest level's communicator
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_boundary = nullptr, ev_comm = nullptr;
  double* halo_lo = nullptr;
  double* halo_hi = nullptr;
  // NVLink peer-store interface sum (elas_set_peer_exchange): my flags (PF_*), the neighbours'
  // IPC-mapped halo buffers and flags, the exchange epoch
  bool peer_on = false;
  unsigned long long peer_epoch = 0;
  unsigned long long* peer_flags = nullptr;
  double* peer_lo_halo = nullptr;           // the lower rank's halo_hi
  double* peer_hi_halo = nullptr;           // the upper rank's halo_lo
  unsigned long long* peer_lo_flags = nullptr;
  unsigned long long* peer_hi_flags = nullptr;
  // measurement hook
  bool prof = false;
  std::vector<cudaEvent_t> prof_ev;   // pairs (start, stop), reused
  size_t prof_used = 0;
  // solver state (elas_solver.cu), allocated on first use
  int qlayout = 0;                    // qdata layout of the variant (QD_LAYOUT_*)
  double* dinv = nullptr;             // cached 1 / diag(A) (elas_diagonal)
  double* red = nullptr;              // reduction partials + device scalars
  double* work = nullptr;             // 4 vectors for elas_pcg (r, z, p, t)
};


struct elas_cheb {
  elas_op* op = nullptr;
  int order = 3;
  double alpha = 0.1, beta = 1.1, lam_max = 0.0;
  double* buf = nullptr;   // r, dv, t (3 vectors)
};

#include <functional>

namespace elas {
void free_solver_state(elas_op* op);
// solver internals shared with elas_gmg.cu (elas_solver.cu)
using PrecondFn = std::function<int(const double* r, double* z)>;
constexpr int PC_CALLBACK = 100;
int cheb_run(elas_cheb* ch, const double* b, double* x, bool x_zero);
// PCG from x = 0; kind: ELAS_PC_NONE / ELAS_PC_JACOBI / PC_CALLBACK (M).  check = false: exactly
// maxit iterations with no host synchronisation (a fixed-length inner solve).
// flexible: Polak-Ribiere beta (flexible CG) for a preconditioner that is not a fixed linear map
// (the V-cycle with a fixed-length inner PCG coarse solve)
int pcg_core(elas_op* op, int kind, const PrecondFn& M, const double* b, double* x, double rtol, int maxit,
             bool check, elas_solve_report* rep, double* history, bool flexible = false);
// exchange the partial interface planes of y with the neighbour ranks and add them (NCCL mode,
// synchronous on the op's stream); no-op for nranks == 1 or external mode
int exchange_planes(elas_op* op, double* y);
// the two halves of exchange_planes around the interior elements (elas_apply)
int exchange_begin(elas_op* op, double* y);
int exchange_end(elas_op* op, double* y);
// peer-mode flags (elas_op::peer_flags): written by the neighbours over NVLink
enum { PF_FILLED_LO = 0, PF_FILLED_HI = 1, PF_CONSUMED_LO = 2, PF_CONSUMED_HI = 3, PF_COUNT = 4 };
// make an external-mode slab op (nranks > 1, no communicator) an NCCL-mode op on a borrowed
// communicator (GMG levels share the finest level's); the op does not destroy it
int attach_comm(elas_op* op, ncclComm_t comm);
// the paper's ablation stages 0 (PA), 1 (+SF), 2 (+Voigt) over elements [e0, e1) (elas_ablation.cu)
cudaError_t ablation_apply(elas_op* op, int stage, const double* x, double* y, int64_t e0, int64_t e1,
                           cudaStream_t st);
}  // namespace elas
