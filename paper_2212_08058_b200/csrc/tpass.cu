// Temporal-pass instantiations (all compiled temporal radii, forward + adjoint).
#include "launch.h"

namespace sfseg {
template <int MODE>
static cudaError_t launch_tpass_t(int RT, const TpassParams& P, int B, cudaStream_t st) {
  dim3 grid((unsigned)((P.frame4 + kTpThreads - 1) / kTpThreads), (unsigned)B);
  switch (RT) {
#define TP_CASE(r)                                             \
  case r:                                                      \
    if (P.halo_lo || P.halo_hi)                                \
      tpass_kernel<r, MODE, true><<<grid, kTpThreads, 0, st>>>(P);    \
    else                                                       \
      tpass_kernel<r, MODE, false><<<grid, kTpThreads, 0, st>>>(P);   \
    return cudaGetLastError();
    TP_CASE(0) TP_CASE(1) TP_CASE(2) TP_CASE(3) TP_CASE(4) TP_CASE(5) TP_CASE(6) TP_CASE(8) TP_CASE(9)
    TP_CASE(12) TP_CASE(16)
#undef TP_CASE
    default:
      return cudaErrorInvalidValue;
  }
}
cudaError_t launch_tpass_fwd(int RT, const TpassParams& P, int B, cudaStream_t st) {
  return launch_tpass_t<TP_FWD>(RT, P, B, st);
}
cudaError_t launch_tpass_fwd16(int RT, const TpassParams& P, int B, cudaStream_t st) {
  return launch_tpass_t<TP_FWD16>(RT, P, B, st);
}
cudaError_t launch_tpass_bwd16(int RT, const TpassParams& P, int B, cudaStream_t st) {
  return launch_tpass_t<TP_BWD16>(RT, P, B, st);
}
cudaError_t launch_tpass_bwd(int RT, const TpassParams& P, int B, cudaStream_t st) {
  return launch_tpass_t<TP_BWD>(RT, P, B, st);
}
cudaError_t launch_tpass_fwdf(int RT, const TpassParams& P, int B, cudaStream_t st) {
  return launch_tpass_t<TP_FWDF>(RT, P, B, st);
}
cudaError_t launch_tpass3(int RT, const Tpass3Params& P, int B, cudaStream_t st, bool f16) {
  dim3 grid((unsigned)((P.frame2 + kTpThreads - 1) / kTpThreads), (unsigned)B);
  switch (RT) {
#define TP3_CASE(r)                                             \
  case r:                                                       \
    if (f16)                                                    \
      tpass3_kernel<r, true><<<grid, kTpThreads, 0, st>>>(P);   \
    else                                                        \
      tpass3_kernel<r, false><<<grid, kTpThreads, 0, st>>>(P);  \
    return cudaGetLastError();
    TP3_CASE(0) TP3_CASE(1) TP3_CASE(2) TP3_CASE(3) TP3_CASE(4) TP3_CASE(5) TP3_CASE(6) TP3_CASE(8) TP3_CASE(9)
    TP3_CASE(12) TP3_CASE(16)
#undef TP3_CASE
    default:
      return cudaErrorInvalidValue;
  }
}
}  // namespace sfseg
