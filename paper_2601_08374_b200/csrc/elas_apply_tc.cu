// Launch wrapper for the FP64 tensor-core (DMMA) kernel, p = 6, q = 8 (elas_apply_tc.cuh).
#include "elas_apply_tc.cuh"

namespace elas {

cudaError_t apply_tc_info(ApplyLaunch* info) {
  info->threads = 32 * tc::WPE * tc::EPC;
  info->elems_per_cta = tc::EPC;
  info->smem_bytes = sizeof(double) * (size_t)tc::EPC * tc::ELEM_SMEM;
  return cudaSuccess;
}

cudaError_t apply_tc_launch(const Slab& s, const double* x, double* y, const double* qd, const double* rr,
                            const double* tables, int64_t e_begin, int64_t e_end, cudaStream_t st) {
  ApplyLaunch L;
  apply_tc_info(&L);
  static KernelPrep prep;   // per device
  int pref = 0;
  cudaError_t e = prep.prep(tc::apply_tc_kernel, L.threads, L.smem_bytes, &pref);
  if (e != cudaSuccess) return e;
  const int64_t ne = e_end - e_begin;
  if (ne <= 0) return cudaSuccess;
  const int64_t nb = (ne + tc::EPC - 1) / tc::EPC;
  const int64_t grid = nb < pref ? nb : pref;   // persistent element slots
  tc::apply_tc_kernel<<<(unsigned)grid, L.threads, L.smem_bytes, st>>>(x, y, qd, rr, tables, s, e_begin, e_end);
  return cudaGetLastError();
}

}  // namespace elas

ELAS_DCHECK_READER(dcheck_tc)
