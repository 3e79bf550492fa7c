// Host-side launchers of the radius-templated pass kernels (one translation
// unit per mode so the heavy instantiations compile in parallel).
#pragma once
#include <cuda_runtime.h>

#include "spass.cuh"
#include "tpass.cuh"
#include "f3d.cuh"

namespace sfseg {
cudaError_t launch_spass_fwd(int R, const SpassParams& P, int grid, cudaStream_t st);
cudaError_t launch_spass_bwd(int R, const SpassParams& P, int grid, cudaStream_t st);
cudaError_t launch_tpass_fwd(int RT, const TpassParams& P, int B, cudaStream_t st);
// TP_FWD16: v written as two fp16 planes for the tcgen05 spatial pass (spass_tc6.cuh)
cudaError_t launch_tpass_fwd16(int RT, const TpassParams& P, int B, cudaStream_t st);
cudaError_t launch_tpass_bwd16(int RT, const TpassParams& P, int B, cudaStream_t st);
cudaError_t launch_tpass_bwd(int RT, const TpassParams& P, int B, cudaStream_t st);
cudaError_t launch_tpass_fwdf(int RT, const TpassParams& P, int B, cudaStream_t st);
// f16: the three outputs as two fp16 planes each (the tcgen05 plain passes; Tpass3Params F16 fields)
cudaError_t launch_tpass3(int RT, const Tpass3Params& P, int B, cudaStream_t st, bool f16 = false);
bool spass_tc_supported(int R);
int spass_tc_occupancy(int R, int fmt = 0);
int spass_tc_boxw(int R);
// fmt 0: three bf16 planes / six products; 1: two fp16 planes / three products (needs the
// preceding temporal pass's per-volume max |v|: TpassParams::vmax -> SpassParams::vslot)
cudaError_t launch_spass_tc(int R, const SpassParams& P, int grid, int fmt, cudaStream_t st);
// tcgen05 / TMEM spatial pass (spass_tc6.cuh): strips of 128 output columns, x-blocks of 128 rows,
// y-blocks of 64 rows; input v as two fp16 planes (TP_FWD16), forward epilogues only
bool spass_tc6_supported(int R);
size_t spass_tc6_smem(int R);
cudaError_t launch_spass_tc6(int R, const SpassParams& P, int grid, cudaStream_t st);
bool f3d_supported(int RT, int R);
int f3d_occupancy(int RT, int R);
cudaError_t launch_f3d(int RT, int R, const F3dParams& P, int grid, cudaStream_t st);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the attribute is
// per device, so a process-wide "done" flag would skip it on the second GPU (sfseg_api.cu).
cudaError_t set_smem_attr_once(const void* kernel, size_t smem);
}  // namespace sfseg
