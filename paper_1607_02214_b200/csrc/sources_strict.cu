// Sources / CFL stencil kernels, strict build (--fmad=false): bit-identical
// to the reference (fast paths replayed exactly, exact re-run of flagged cells).
#include "sources_launch.inc"
