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
//   [63:52] step (relative to the last reset)  [51:49] step phase (execution
//   order within the step)  [48:47] sweep axis  [46:0] phase-specific
//   position (see the kernels), whose low 2 bits are the error kind.
// Sweep positions are pencil << 20 | sub << 19 | zone << 2 | kind: pencils
// per face < 2^27 and strip positions < 2^17, checked when a block is
// created (kMaxPencils / kMaxStrip); a run checks its errors at least every
// kMaxStepsPerCheck steps so the step field never wraps.
enum : unsigned long long { kNoError = ~0ull };
enum StepPhase : int { kPhaseCfl = 0, kPhaseSweep0 = 1, kPhaseSweep1 = 2, kPhaseSweep2 = 3,
                       kPhaseSources = 4 };
enum ErrKind : int { kErrStepRejected = 0, kErrLagUnphysical = 1, kErrDensity = 2,
                     kErrPressure = 3 };
constexpr int kErrStepShift = 52, kErrPhaseShift = 49, kErrAxisShift = 47, kErrPosBits = 47;
constexpr unsigned long long kErrStepMask = (1ull << (64 - kErrStepShift)) - 1;
constexpr unsigned long long kErrPosMask = (1ull << kErrPosBits) - 1;
constexpr long kMaxStepsPerCheck = (long)kErrStepMask - 1;  // the next step's CFL uses +1
constexpr unsigned long long kMaxPencils = 1ull << (kErrPosBits - 20);
constexpr int kMaxStrip = 1 << 17;

PPMLR_HD unsigned long long err_key(unsigned long long step, int phase, int axis,
                                    unsigned long long pos) {
  return ((step & kErrStepMask) << kErrStepShift) |
         ((unsigned long long)phase << kErrPhaseShift) |
         ((unsigned long long)axis << kErrAxisShift) | (pos & kErrPosMask);
}
PPMLR_HD int err_phase(unsigned long long key) { return (int)((key >> kErrPhaseShift) & 7); }
PPMLR_HD int err_axis(unsigned long long key) { return (int)((key >> kErrAxisShift) & 3); }
PPMLR_HD unsigned long long err_step(unsigned long long key) { return key >> kErrStepShift; }
PPMLR_HD unsigned long long err_pos(unsigned long long key) { return key & kErrPosMask; }

}  // namespace ppmlr_b200
