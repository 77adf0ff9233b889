// Strict sweep: compiled with --fmad=false; bit-identical to the reference.
#define PPMLR_KNS strict
#ifndef PPMLR_SWEEP_V2_ON
#define PPMLR_SWEEP_V2_ON 1  // sweep_v2.cuh schedule (same operation order) for the compile-time tile
#endif
#ifndef PPMLR_SWEEP_V2_DIPOLE
#define PPMLR_SWEEP_V2_DIPOLE 1
#endif
#define PPMLR_LAUNCH_NAME launch_sweep_strict
#include "sweep_launch.inc"
