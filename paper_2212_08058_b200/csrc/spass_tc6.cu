// tcgen05 spatial-pass instantiations (spass_tc6.cuh) + launcher.
#include "launch.h"
#include "spass_tc6.cuh"

namespace sfseg {
namespace {
template <int R, int EPI>
cudaError_t launch_tc6_epi(const SpassParams& P, int grid, cudaStream_t st) {
  const size_t smem = t6_smem_bytes(R);
  cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(spass_tc6_kernel<R, EPI>), smem);
  if (e != cudaSuccess) return e;
  spass_tc6_kernel<R, EPI><<<grid, k6Threads, smem, st>>>(P);
  return cudaGetLastError();
}
template <int R>
cudaError_t launch_tc6_one(const SpassParams& P, int grid, cudaStream_t st) {
  if (P.plain) return launch_tc6_epi<R, EPI_PLAIN>(P, grid, st);
  if (P.tape_u || P.pprev) return launch_tc6_epi<R, EPI_FWD_OPT>(P, grid, st);
  return launch_tc6_epi<R, EPI_FWD>(P, grid, st);
}
}  // namespace

#define T6_RADII(X) X(8) X(9) X(12) X(16) X(18) X(24) X(32) X(36)

bool spass_tc6_supported(int R) {
  switch (R) {
#define T6_SUP(r) case r:
    T6_RADII(T6_SUP)
#undef T6_SUP
    return true;
    default:
      return false;
  }
}
size_t spass_tc6_smem(int R) { return t6_smem_bytes(R); }
cudaError_t launch_spass_tc6(int R, const SpassParams& P, int grid, cudaStream_t st) {
  switch (R) {
#define T6_CASE(r) \
  case r:          \
    return launch_tc6_one<r>(P, grid, st);
    T6_RADII(T6_CASE)
#undef T6_CASE
    default:
      return cudaErrorInvalidValue;
  }
}
}  // namespace sfseg
