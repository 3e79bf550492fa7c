// Megakernel instantiations (the (r_s, r_t) pairs of the large-radius configs) + launcher.
#include "launch.h"
#include "mk.cuh"

namespace sfseg {
namespace {
template <int R, int RT>
cudaError_t mk_one(const MkParams& P, int* grid_out, cudaStream_t st, bool launch) {
  const size_t smem = mk_smem_bytes(R, RT);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(mk_kernel<R, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  int per_sm = 0, dev = 0, sms = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mk_kernel<R, RT>, kMkThreads, smem);
  if (e != cudaSuccess) return e;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  *grid_out = per_sm * sms;  // every CTA resident: the spin-waits cannot deadlock
  if (!launch) return cudaSuccess;
  mk_kernel<R, RT><<<*grid_out, kMkThreads, smem, st>>>(P);
  return cudaGetLastError();
}
}  // namespace

bool mk_supported(int RT, int R) { return (R == 24 && RT == 6) || (R == 18 && RT == 5) || (R == 36 && RT == 9); }

cudaError_t launch_mk(int RT, int R, const MkParams& P, int* grid_out, cudaStream_t st, bool launch) {
  if (R == 24 && RT == 6) return mk_one<24, 6>(P, grid_out, st, launch);
  if (R == 18 && RT == 5) return mk_one<18, 5>(P, grid_out, st, launch);
  if (R == 36 && RT == 9) return mk_one<36, 9>(P, grid_out, st, launch);
  return cudaErrorInvalidValue;
}
}  // namespace sfseg
