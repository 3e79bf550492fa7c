// Forward spatial-pass instantiations (all compiled radii).
#define SPASS_MODE SP_FWD
#define SPASS_FN launch_spass_fwd
#include "spass_launch.inc"
