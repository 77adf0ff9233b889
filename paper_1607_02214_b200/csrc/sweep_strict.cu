// Strict sweep: compiled with --fmad=false; bit-identical to the reference.
#define PPMLR_KNS strict
#define PPMLR_LAUNCH_NAME launch_sweep_strict
#include "sweep_launch.inc"
