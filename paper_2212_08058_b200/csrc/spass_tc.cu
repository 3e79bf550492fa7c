// Tensor-core forward spatial-pass instantiations (spass_tc.cuh).
#include "launch.h"
#include "spass_tc.cuh"

namespace sfseg {
namespace {
template <int R, int EPI, int FMT>
cudaError_t launch_tc_epi(const SpassParams& P, int grid, cudaStream_t st) {
  const size_t smem = sptc_smem_bytes(R, FMT);
  cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(spass_tc_kernel<R, EPI, FMT>), smem);
  if (e != cudaSuccess) return e;
  spass_tc_kernel<R, EPI, FMT><<<grid, kSpassThreads, smem, st>>>(P);
  return cudaGetLastError();
}
template <int R>
cudaError_t launch_tc_one(const SpassParams& P, int grid, int fmt, cudaStream_t st) {
  if (P.full_epi) return fmt ? launch_tc_epi<R, EPI_FULL, 1>(P, grid, st) : launch_tc_epi<R, EPI_FULL, 0>(P, grid, st);
  if (P.plain) return fmt ? launch_tc_epi<R, EPI_PLAIN, 1>(P, grid, st) : launch_tc_epi<R, EPI_PLAIN, 0>(P, grid, st);
  if (fmt) {
    if (P.tape_u || P.pprev) return launch_tc_epi<R, EPI_FWD_OPT, 1>(P, grid, st);
    return launch_tc_epi<R, EPI_FWD, 1>(P, grid, st);
  }
  if (P.tape_u || P.pprev) return launch_tc_epi<R, EPI_FWD_OPT, 0>(P, grid, st);
  return launch_tc_epi<R, EPI_FWD, 0>(P, grid, st);
}
}  // namespace

#define SPTC_RADII(X) X(8) X(9) X(12) X(16) X(18) X(24) X(32) X(36) X(48)

bool spass_tc_supported(int R) {
  switch (R) {
#define TC_SUP(r) case r:
    SPTC_RADII(TC_SUP)
#undef TC_SUP
    return true;
    default:
      return false;
  }
}
int spass_tc_occupancy(int R, int fmt) {
  switch (R) {
#define TC_OCC(r) \
  case r:         \
    return sptc_ctas_per_sm(r, fmt);
    SPTC_RADII(TC_OCC)
#undef TC_OCC
    default:
      return 1;
  }
}
int spass_tc_boxw(int R) {
  switch (R) {
#define TC_BW(r) \
  case r:        \
    return sptc_boxw(r);
    SPTC_RADII(TC_BW)
#undef TC_BW
    default:
      return 0;
  }
}
cudaError_t launch_spass_tc(int R, const SpassParams& P, int grid, int fmt, cudaStream_t st) {
  switch (R) {
#define TC_CASE(r) \
  case r:          \
    return launch_tc_one<r>(P, grid, fmt, st);
    SPTC_RADII(TC_CASE)
#undef TC_CASE
    default:
      return cudaErrorInvalidValue;
  }
}
}  // namespace sfseg
