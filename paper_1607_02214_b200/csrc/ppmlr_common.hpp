// Host/device-common definitions of the hot path: run constants, strip
// slots and the first-failure error-key layout.
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define PPMLR_HD __host__ __device__ __forceinline__
#else
#define PPMLR_HD inline
#endif

namespace ppmlr_b200 {

constexpr int kG = 4;  // device ghost width (the dependency window)

struct Consts {
  double gamma, mu0, pressure_floor;
  double gm1;      // gamma - 1.0   (hoisted; same rounding as the reference's inline form)
  double two_mu0;  // 2.0 * mu0     (hoisted; exact)
  // rcp_refined of gm1, two_mu0, mu0, 6 and 3 (the divisor-only half of
  // nvcc's `/`), computed once on the device when the block is created
  double r_gm1, r_two_mu0, r_mu0, r6, r3;
};

// Strip-frame variable slots (proj/include/ppmlr/ppm1d.hpp:50).
enum : int { kRho = 0, kUn, kUt1, kUt2, kBn, kBt1, kBt2, kPE };

// Error words: one 64-bit key per block, atomicMin'd, so the first failure in
// the reference's loop order wins.  Layout (high to low):
//   [63:46] step (relative to the last reset)  [45:43] step phase (execution
//   order within the step)  [42:41] sweep axis  [40:0] phase-specific
//   position (see the kernels), whose low 2 bits are the error kind.
enum : unsigned long long { kNoError = ~0ull };
enum StepPhase : int { kPhaseCfl = 0, kPhaseSweep0 = 1, kPhaseSweep1 = 2, kPhaseSweep2 = 3,
                       kPhaseSources = 4 };
enum ErrKind : int { kErrStepRejected = 0, kErrLagUnphysical = 1, kErrDensity = 2,
                     kErrPressure = 3 };

PPMLR_HD unsigned long long err_key(unsigned long long step,
                                                               int phase, int axis,
                                                               unsigned long long pos) {
  return ((step & 0x3FFFFull) << 46) | ((unsigned long long)phase << 43) |
         ((unsigned long long)axis << 41) | (pos & ((1ull << 41) - 1));
}

}  // namespace ppmlr_b200
