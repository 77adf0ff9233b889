// Device-side per-cell algebra of the PPMLR-MHD hot path (sm_100a, FP64).
//
// Every helper here keeps the reference's IEEE-754 operation order
// (C++ left-to-right association) so that, compiled with --fmad=false, the
// device results are bit-identical to the reference CPU implementation.
// The fast build (--fmad=true, PPMLR_FAST_MATH) may contract and fold.
// Citations are to /root/reference/proj.
#pragma once
#include <cstdint>

#ifndef PPMLR_KNS
#define PPMLR_KNS strict
#endif

namespace ppmlr_b200 {

struct Consts {
  double gamma, mu0, pressure_floor;
  double gm1;      // gamma - 1.0   (hoisted; same rounding as the reference's inline form)
  double two_mu0;  // 2.0 * mu0     (hoisted; exact)
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

__host__ __device__ __forceinline__ unsigned long long err_key(unsigned long long step,
                                                               int phase, int axis,
                                                               unsigned long long pos) {
  return ((step & 0x3FFFFull) << 46) | ((unsigned long long)phase << 43) |
         ((unsigned long long)axis << 41) | (pos & ((1ull << 41) - 1));
}

namespace PPMLR_KNS {

// std::min / std::max / std::clamp argument-order semantics.
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double sclamp(double v, double lo, double hi) {
  return (v < lo) ? lo : ((hi < v) ? hi : v);
}

// physics.cpp:63-72 fast_speed: total field b = B' + bd, |b|^2 in xyz order.
template <int DIR>
__device__ __forceinline__ double fast_speed3(const double* s, double bdx, double bdy,
                                              double bdz, const Consts& c) {
  const double b0 = s[4] + bdx, b1 = s[5] + bdy, b2 = s[6] + bdz;
  const double bdir = DIR == 0 ? b0 : (DIR == 1 ? b1 : b2);
  const double a2 = (c.gamma * s[7]) / s[0];
  const double ca2 = ((b0 * b0 + b1 * b1) + b2 * b2) / (c.mu0 * s[0]);
  const double can2 = (bdir * bdir) / (c.mu0 * s[0]);
  const double sum = a2 + ca2;
  const double disc = sqrt(smax(0.0, sum * sum - (4.0 * a2) * can2));
  return sqrt(0.5 * (sum + disc));
}

// ppm1d.cpp:29-37 fast_speed_strip: |b|^2 in strip order.
__device__ __forceinline__ double fast_speed_strip(double rho, double p, double btn,
                                                   double btt1, double btt2, const Consts& c) {
  const double a2 = (c.gamma * p) / rho;
  const double ca2 = ((btn * btn + btt1 * btt1) + btt2 * btt2) / (c.mu0 * rho);
  const double can2 = (btn * btn) / (c.mu0 * rho);
  const double sum = a2 + ca2;
  const double disc = sqrt(smax(0.0, sum * sum - (4.0 * a2) * can2));
  return sqrt(0.5 * (sum + disc));
}

// ppm1d.cpp:39-52 prim_to_cons_strip; only the energy slot is non-trivial.
__device__ __forceinline__ double strip_energy(const double* w, const Consts& c) {
  return (w[kPE] / c.gm1 + (0.5 * w[kRho]) * ((w[kUn] * w[kUn] + w[kUt1] * w[kUt1]) +
                                               w[kUt2] * w[kUt2])) +
         ((w[kBn] * w[kBn] + w[kBt1] * w[kBt1]) + w[kBt2] * w[kBt2]) / c.two_mu0;
}

// physics.cpp:29-37 prim_to_cons (xyz order) into u[8].
__device__ __forceinline__ void prim_to_cons3(const double* s, double* u, const Consts& c) {
  u[0] = s[0];
  u[1] = s[1] * s[0];
  u[2] = s[2] * s[0];
  u[3] = s[3] * s[0];
  u[4] = s[4];
  u[5] = s[5];
  u[6] = s[6];
  const double v2 = (s[1] * s[1] + s[2] * s[2]) + s[3] * s[3];
  const double b2 = (s[4] * s[4] + s[5] * s[5]) + s[6] * s[6];
  u[7] = (s[7] / c.gm1 + (0.5 * s[0]) * v2) + b2 / c.two_mu0;
}

// physics.cpp:39-57 cons_to_prim (xyz order).  Returns 0 ok, 1 density, 2 pressure.
__device__ __forceinline__ int cons_to_prim3(const double* u, double* q, const Consts& c) {
  if (!(u[0] > 0.0)) return 1;
  q[0] = u[0];
  q[1] = u[1] / u[0];
  q[2] = u[2] / u[0];
  q[3] = u[3] / u[0];
  q[4] = u[4];
  q[5] = u[5];
  q[6] = u[6];
  const double m2 = (u[1] * u[1] + u[2] * u[2]) + u[3] * u[3];
  const double b2 = (u[4] * u[4] + u[5] * u[5]) + u[6] * u[6];
  const double internal = (u[7] - (0.5 * m2) / u[0]) - b2 / c.two_mu0;
  q[7] = c.gm1 * internal;
  if (!(q[7] > 0.0)) {
    if (c.pressure_floor > 0.0)
      q[7] = c.pressure_floor;
    else
      return 2;
  }
  return 0;
}

// ppm1d.cpp:14-24 limited_slope with hoisted geometry:
//   c0 = dx_k/((dx_{k-1}+dx_k)+dx_{k+1}), A = (2dx_{k-1}+dx_k)/(dx_{k+1}+dx_k),
//   B = (dx_k+2dx_{k+1})/(dx_{k-1}+dx_k)   (bit-exact: same subexpressions).
__device__ __forceinline__ double limited_slope(double qm, double q0, double qp, double c0,
                                                double A, double B) {
  const double dql = q0 - qm;
  const double dqr = qp - q0;
  if (dqr * dql <= 0.0) return 0.0;
  const double dq = c0 * (A * dqr + B * dql);
  const double lim = 2.0 * smin(fabs(dql), fabs(dqr));
  return copysign(smin(fabs(dq), lim), dq);
}

// ppm1d.cpp:217-224 CW84 interface value at edge m (i = m-1) with hoisted e0..e4.
__device__ __forceinline__ double interface_value(double qi, double qi1, double dmi,
                                                  double dmi1, const double* e) {
  const double dqr = qi1 - qi;
  return (qi + e[0] * dqr) + e[1] * ((e[2] * dqr - e[3] * dmi1) + e[4] * dmi);
}

// ppm1d.cpp:232-246 monotonicity limiter.  In: al, ar (interface values), av.
// Out: al, ar limited, six.
__device__ __forceinline__ void limit_parabola(double& al, double& ar, double av, double& six) {
  if ((ar - av) * (av - al) <= 0.0) {
    al = ar = av;
  } else {
    const double d = ar - al;
    const double t = d * (av - 0.5 * (al + ar));
    if (t > (d * d) / 6.0)
      al = 3.0 * av - 2.0 * ar;
    else if (t < ((-d) * d) / 6.0)
      ar = 3.0 * av - 2.0 * al;
  }
  six = 6.0 * (av - 0.5 * (al + ar));
}

// ppm1d.hpp:20-26 parabola means; hs = 0.5*sigma, tw = 1.0 - (2.0*sigma)/3.0 are
// shared by every variable with the same sigma (common-subexpression, exact).
__device__ __forceinline__ double avg_left(double l, double r, double six, double hs,
                                           double tw) {
  return l + hs * ((r - l) + tw * six);
}
__device__ __forceinline__ double avg_right(double l, double r, double six, double hs,
                                            double tw) {
  return r - hs * ((r - l) - tw * six);
}

// ppm1d.cpp:69-109 solve_edge + edge_flux.  ql/qr strip-frame traced states,
// bl/br total-field offsets (bd components in strip order a, b, d).
__device__ __forceinline__ double solve_edge(const double* ql, const double* qr,
                                             const double* bl, const double* br,
                                             const Consts& c, double* f) {
  const double wl = ql[kRho] * fast_speed_strip(ql[kRho], ql[kPE], ql[kBn] + bl[0],
                                                ql[kBt1] + bl[1], ql[kBt2] + bl[2], c);
  const double wr = qr[kRho] * fast_speed_strip(qr[kRho], qr[kPE], qr[kBn] + br[0],
                                                qr[kBt1] + br[1], qr[kBt2] + br[2], c);
  const double pl =
      ql[kPE] + ((ql[kBt1] * ql[kBt1] + ql[kBt2] * ql[kBt2]) - ql[kBn] * ql[kBn]) / c.two_mu0;
  const double pr =
      qr[kPE] + ((qr[kBt1] * qr[kBt1] + qr[kBt2] * qr[kBt2]) - qr[kBn] * qr[kBn]) / c.two_mu0;
  const double wsum = wl + wr;
  const double ustar = (((wl * ql[kUn] + wr * qr[kUn]) + pl) - pr) / wsum;
  const double pstar = ((wr * pl + wl * pr) + (wl * wr) * (ql[kUn] - qr[kUn])) / wsum;
  const double bn = 0.5 * (ql[kBn] + qr[kBn]);
  const double s = bn < 0.0 ? -1.0 : 1.0;
  const double al = 1.0 / sqrt(c.mu0 * ql[kRho]);
  const double ar = 1.0 / sqrt(c.mu0 * qr[kRho]);
  const double asum = al + ar;
  const double bt1 = ((s * (qr[kUt1] - ql[kUt1]) + ar * qr[kBt1]) + al * ql[kBt1]) / asum;
  const double bt2 = ((s * (qr[kUt2] - ql[kUt2]) + ar * qr[kBt2]) + al * ql[kBt2]) / asum;
  const double vt1 = ql[kUt1] + (s * al) * (bt1 - ql[kBt1]);
  const double vt2 = ql[kUt2] + (s * al) * (bt2 - ql[kBt2]);
  f[kRho] = 0.0;
  f[kUn] = pstar;
  f[kUt1] = ((-bn) * bt1) / c.mu0;
  f[kUt2] = ((-bn) * bt2) / c.mu0;
  f[kBn] = (-ustar) * bn;
  f[kBt1] = (-bn) * vt1;
  f[kBt2] = (-bn) * vt2;
  f[kPE] = pstar * ustar - (bn * (vt1 * bt1 + vt2 * bt2)) / c.mu0;
  return ustar;
}

}  // namespace PPMLR_KNS
}  // namespace ppmlr_b200
