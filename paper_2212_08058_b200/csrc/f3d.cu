// Fused single-pass 3D iteration (small radii) instantiations + launcher.
#include "f3d.cuh"
#include "launch.h"

namespace sfseg {
namespace {
template <int RT, int R, bool OPT>
cudaError_t f3d_launch_opt(const F3dParams& P, int grid, cudaStream_t st) {
  const size_t smem = f3d_smem_bytes(RT, R);
  cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(f3d_kernel<RT, R, OPT>), smem);
  if (e != cudaSuccess) return e;
  f3d_kernel<RT, R, OPT><<<grid, kF3dThreads, smem, st>>>(P);
  return cudaGetLastError();
}
template <int RT, int R>
cudaError_t f3d_launch_one(const F3dParams& P, int grid, cudaStream_t st) {
  return (P.tape_u || P.rayleigh) ? f3d_launch_opt<RT, R, true>(P, grid, st) : f3d_launch_opt<RT, R, false>(P, grid, st);
}
template <int RT>
cudaError_t f3d_launch_rt(int R, const F3dParams& P, int grid, cudaStream_t st) {
  switch (R) {
    case 1: return f3d_launch_one<RT, 1>(P, grid, st);
    case 2: return f3d_launch_one<RT, 2>(P, grid, st);
    case 3: return f3d_launch_one<RT, 3>(P, grid, st);
    case 4: return f3d_launch_one<RT, 4>(P, grid, st);
    case 5: return f3d_launch_one<RT, 5>(P, grid, st);
    case 6: return f3d_launch_one<RT, 6>(P, grid, st);
    case 8: return f3d_launch_one<RT, 8>(P, grid, st);
    default: return cudaErrorInvalidValue;
  }
}
template <int RT>
int f3d_occ_rt(int R) {
  switch (R) {
    case 1: return f3d_ctas_per_sm(RT, 1);
    case 2: return f3d_ctas_per_sm(RT, 2);
    case 3: return f3d_ctas_per_sm(RT, 3);
    case 4: return f3d_ctas_per_sm(RT, 4);
    case 5: return f3d_ctas_per_sm(RT, 5);
    case 6: return f3d_ctas_per_sm(RT, 6);
    case 8: return f3d_ctas_per_sm(RT, 8);
    default: return 1;
  }
}
}  // namespace

bool f3d_supported(int RT, int R) {
  return RT >= 0 && RT <= kF3dMaxRT && (R == 1 || R == 2 || R == 3 || R == 4 || R == 5 || R == 6 || R == 8);
}
int f3d_occupancy(int RT, int R) {
  switch (RT) {
    case 0: return f3d_occ_rt<0>(R);
    case 1: return f3d_occ_rt<1>(R);
    case 2: return f3d_occ_rt<2>(R);
    default: return f3d_occ_rt<3>(R);
  }
}
cudaError_t launch_f3d(int RT, int R, const F3dParams& P, int grid, cudaStream_t st) {
  switch (RT) {
    case 0: return f3d_launch_rt<0>(R, P, grid, st);
    case 1: return f3d_launch_rt<1>(R, P, grid, st);
    case 2: return f3d_launch_rt<2>(R, P, grid, st);
    case 3: return f3d_launch_rt<3>(R, P, grid, st);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace sfseg
