// Backward (adjoint) spatial-pass instantiations (all compiled radii).
#define SPASS_MODE SP_BWD
#define SPASS_FN launch_spass_bwd
#include "spass_launch.inc"
