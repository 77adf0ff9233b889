// Fast sweep: compiled with --fmad=true and PPMLR_FAST_MATH (reciprocal folding);
// gated by the tolerance in DESIGN.md / tests/test_gpu_parity.py.
#define PPMLR_FAST_MATH 1
#ifndef PPMLR_FAST_SQRT_RSQ
#define PPMLR_FAST_SQRT_RSQ 1  // sqrt as x * rsqrt(x) (exact_div.cuh)
#endif
#define PPMLR_KNS fast
#ifndef PPMLR_SWEEP_V2_ON
#define PPMLR_SWEEP_V2_ON 1  // sweep_v2.cuh schedule for the compile-time tile
#endif
#ifndef PPMLR_SWEEP_V2_DIPOLE
#define PPMLR_SWEEP_V2_DIPOLE 1  // ... with the dipole too (B_d read from global memory)
#endif
#define PPMLR_LAUNCH_NAME launch_sweep_fast
#include "sweep_launch.inc"
