// Host-side launchers of the radius-templated pass kernels (one translation
// unit per mode so the heavy instantiations compile in parallel).
#pragma once
#include <cuda_runtime.h>

#include "spass.cuh"
#include "tpass.cuh"
#include "f3d.cuh"
#include "mk.cuh"

namespace sfseg {
cudaError_t launch_spass_fwd(int R, const SpassParams& P, int grid, cudaStream_t st);
cudaError_t launch_spass_bwd(int R, const SpassParams& P, int grid, cudaStream_t st);
cudaError_t launch_tpass_fwd(int RT, const TpassParams& P, int B, cudaStream_t st);
cudaError_t launch_tpass_bwd(int RT, const TpassParams& P, int B, cudaStream_t st);
cudaError_t launch_tpass_fwdf(int RT, const TpassParams& P, int B, cudaStream_t st);
bool spass_tc_supported(int R);
int spass_tc_occupancy(int R);
int spass_tc_boxw(int R);
cudaError_t launch_spass_tc(int R, const SpassParams& P, int grid, cudaStream_t st);
bool f3d_supported(int RT, int R);
int f3d_occupancy(int RT, int R);
cudaError_t launch_f3d(int RT, int R, const F3dParams& P, int grid, cudaStream_t st);
bool mk_supported(int RT, int R);
cudaError_t launch_mk(int RT, int R, const MkParams& P, int* grid_out, cudaStream_t st, bool launch);
}  // namespace sfseg
