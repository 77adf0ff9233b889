// Sources / CFL stencil kernels, fast build (--fmad=true, FastMathOps).
#define PPMLR_FAST_MATH 1
#define PPMLR_KNS fast
#define PPMLR_SRC_LAUNCH_NAME launch_sources_fast
#include "sources_launch.inc"
