// tcgen05 spatial-pass instantiations (spass_tc5.cuh) + launcher.
#include "launch.h"
#include "spass_tc5.cuh"

namespace sfseg {
namespace {
template <int R, int EPI>
cudaError_t launch_tc5_epi(const SpassParams& P, int grid, cudaStream_t st) {
  const size_t smem = t5_smem_bytes(R);
  cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(spass_tc5_kernel<R, EPI>), smem);
  if (e != cudaSuccess) return e;
  spass_tc5_kernel<R, EPI><<<grid, k5Threads, smem, st>>>(P);
  return cudaGetLastError();
}
template <int R>
cudaError_t launch_tc5_one(const SpassParams& P, int grid, cudaStream_t st) {
  if (P.plain) return launch_tc5_epi<R, EPI_PLAIN>(P, grid, st);
  if (P.tape_u || P.pprev) return launch_tc5_epi<R, EPI_FWD_OPT>(P, grid, st);
  return launch_tc5_epi<R, EPI_FWD>(P, grid, st);
}
}  // namespace

#define T5_RADII(X) X(8) X(9) X(12) X(16) X(18) X(24)

bool spass_tc5_supported(int R) {
  switch (R) {
#define T5_SUP(r) case r:
    T5_RADII(T5_SUP)
#undef T5_SUP
    return true;
    default:
      return false;
  }
}
cudaError_t launch_spass_tc5(int R, const SpassParams& P, int grid, cudaStream_t st) {
  switch (R) {
#define T5_CASE(r) \
  case r:          \
    return launch_tc5_one<r>(P, grid, st);
    T5_RADII(T5_CASE)
#undef T5_CASE
    default:
      return cudaErrorInvalidValue;
  }
}
}  // namespace sfseg
