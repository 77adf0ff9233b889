// Device-side per-cell algebra of the PPMLR-MHD hot path (sm_100a, FP64).
//
// Every helper here keeps the reference's IEEE-754 operation order
// (C++ left-to-right association) so that, compiled with --fmad=false, the
// device results are bit-identical to the reference CPU implementation.
// The fast build (--fmad=true, PPMLR_FAST_MATH) may contract and fold.
// Citations are to /root/reference/proj.
#pragma once
#include <cstdint>

#include "exact_div.cuh"
#include "ppmlr_common.hpp"

#ifndef PPMLR_KNS
#define PPMLR_KNS strict
#endif

// Fast-build algebra switches (tuning; each measured on the B200)
#ifndef PPMLR_FAST_TRACED
#define PPMLR_FAST_TRACED 0     // fused limiter + parabola means (traced_lr)
#endif
#ifndef PPMLR_FAST_SLOPE_SIGN
#define PPMLR_FAST_SLOPE_SIGN 1 // limited_slope's product test on the sign bits
#endif
#ifndef PPMLR_FAST_RCP_SHARE
#define PPMLR_FAST_RCP_SHARE 1  // one 1/rho per signal speed, rsqrt for 1/sqrt(mu0 rho)
#endif

namespace ppmlr_b200 {

namespace PPMLR_KNS {

// Reciprocals of the run constants and of the literal divisors 6 and 3
// (precomputed per block with rcp_refined; see Consts).
struct KC {
  Consts c;
  double r_gm1, r_two_mu0, r_mu0, r6, r3;
};
__device__ __forceinline__ KC make_kc(const Consts& c) {
  KC k;
  k.c = c;
  k.r_gm1 = c.r_gm1;
  k.r_two_mu0 = c.r_two_mu0;
  k.r_mu0 = c.r_mu0;
  k.r6 = c.r6;
  k.r3 = c.r3;
  return k;
}

// std::min / std::max / std::clamp argument-order semantics.
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double sclamp(double v, double lo, double hi) {
  return (v < lo) ? lo : ((hi < v) ? hi : v);
}

// physics.cpp:63-72 fast_speed: total field b = B' + bd, |b|^2 in xyz order.
// BD = false: no dipole (the total field is B' itself; no `+ 0.0`).
template <int DIR, class Ops, bool BD = true>
__device__ __forceinline__ double fast_speed3(const double* s, double bdx, double bdy,
                                              double bdz, const KC& k, Ops& o) {
  const double b0 = BD ? s[4] + bdx : s[4], b1 = BD ? s[5] + bdy : s[5],
               b2 = BD ? s[6] + bdz : s[6];
  const double bdir = DIR == 0 ? b0 : (DIR == 1 ? b1 : b2);
  double a2, ca2, can2;
  if constexpr (Ops::kFastMath && PPMLR_FAST_RCP_SHARE) {
    // one reciprocal: 1/(mu0 rho) = (1/mu0)(1/rho)
    const double r_rho = o.rcp(s[0]);
    const double r_mr = k.r_mu0 * r_rho;
    a2 = (k.c.gamma * s[7]) * r_rho;
    ca2 = ((b0 * b0 + b1 * b1) + b2 * b2) * r_mr;
    can2 = (bdir * bdir) * r_mr;
  } else {
    const double mr = k.c.mu0 * s[0];
    const double r_mr = o.rcp(mr);
    a2 = o.dv(k.c.gamma * s[7], s[0]);
    ca2 = o.div((b0 * b0 + b1 * b1) + b2 * b2, mr, r_mr);
    can2 = o.div(bdir * bdir, mr, r_mr);
  }
  const double sum = a2 + ca2;
  const double disc = o.sq(smax(0.0, sum * sum - (4.0 * a2) * can2));
  return o.sq(0.5 * (sum + disc));
}

// fast_speed3 for the three directions at once (compute_dt,
// stepper.cpp:128-137): a2, ca2, sum, sum*sum and 4*a2 do not depend on the
// direction, so they are evaluated once (identical operands -> identical
// bits).
template <class Ops>
__device__ __forceinline__ void fast_speed3_all(const double* s, double bdx, double bdy,
                                                double bdz, const KC& k, Ops& o, double* cf) {
  const double b0 = s[4] + bdx, b1 = s[5] + bdy, b2 = s[6] + bdz;
  double a2, ca2, r_mr, mr = 0.0;
  if constexpr (Ops::kFastMath && PPMLR_FAST_RCP_SHARE) {
    const double r_rho = o.rcp(s[0]);
    r_mr = k.r_mu0 * r_rho;
    a2 = (k.c.gamma * s[7]) * r_rho;
    ca2 = ((b0 * b0 + b1 * b1) + b2 * b2) * r_mr;
  } else {
    mr = k.c.mu0 * s[0];
    r_mr = o.rcp(mr);
    a2 = o.dv(k.c.gamma * s[7], s[0]);
    ca2 = o.div((b0 * b0 + b1 * b1) + b2 * b2, mr, r_mr);
  }
  const double sum = a2 + ca2;
  const double ss = sum * sum;
  const double a4 = 4.0 * a2;
  const double bb[3] = {b0, b1, b2};
#pragma unroll
  for (int dir = 0; dir < 3; ++dir) {
    const double can2 = o.div(bb[dir] * bb[dir], mr, r_mr);
    const double disc = o.sq(smax(0.0, ss - a4 * can2));
    cf[dir] = o.sq(0.5 * (sum + disc));
  }
}

// ppm1d.cpp:29-37 fast_speed_strip: |b|^2 in strip order.
template <class Ops>
__device__ __forceinline__ double fast_speed_strip(double rho, double p, double btn,
                                                   double btt1, double btt2, const KC& k,
                                                   Ops& o) {
  double a2, ca2, can2;
  if constexpr (Ops::kFastMath && PPMLR_FAST_RCP_SHARE) {
    const double r_rho = o.rcp(rho);
    const double r_mr = k.r_mu0 * r_rho;
    a2 = (k.c.gamma * p) * r_rho;
    const double bn2 = btn * btn;
    ca2 = ((bn2 + btt1 * btt1) + btt2 * btt2) * r_mr;
    can2 = bn2 * r_mr;
  } else {
    const double mr = k.c.mu0 * rho;
    const double r_mr = o.rcp(mr);
    a2 = o.dv(k.c.gamma * p, rho);
    ca2 = o.div((btn * btn + btt1 * btt1) + btt2 * btt2, mr, r_mr);
    can2 = o.div(btn * btn, mr, r_mr);
  }
  const double sum = a2 + ca2;
  const double disc = o.sq(smax(0.0, sum * sum - (4.0 * a2) * can2));
  return o.sq(0.5 * (sum + disc));
}

// ppm1d.cpp:39-52 prim_to_cons_strip; only the energy slot is non-trivial.
template <class Ops>
__device__ __forceinline__ double strip_energy(const double* w, const KC& k, Ops& o) {
  return (o.div(w[kPE], k.c.gm1, k.r_gm1) +
          (0.5 * w[kRho]) * ((w[kUn] * w[kUn] + w[kUt1] * w[kUt1]) + w[kUt2] * w[kUt2])) +
         o.div((w[kBn] * w[kBn] + w[kBt1] * w[kBt1]) + w[kBt2] * w[kBt2], k.c.two_mu0,
               k.r_two_mu0);
}

// physics.cpp:29-37 prim_to_cons (xyz order) into u[8].
template <class Ops>
__device__ __forceinline__ void prim_to_cons3(const double* s, double* u, const KC& k, Ops& o) {
  u[0] = s[0];
  u[1] = s[1] * s[0];
  u[2] = s[2] * s[0];
  u[3] = s[3] * s[0];
  u[4] = s[4];
  u[5] = s[5];
  u[6] = s[6];
  const double v2 = (s[1] * s[1] + s[2] * s[2]) + s[3] * s[3];
  const double b2 = (s[4] * s[4] + s[5] * s[5]) + s[6] * s[6];
  u[7] = (o.div(s[7], k.c.gm1, k.r_gm1) + (0.5 * s[0]) * v2) +
         o.div(b2, k.c.two_mu0, k.r_two_mu0);
}

// physics.cpp:39-57 cons_to_prim (xyz order), branch-free.  Returns 0 ok,
// 1 non-positive density, 2 non-positive pressure (q is then unspecified).
template <class Ops>
__device__ __forceinline__ int cons_to_prim3(const double* u, double* q, const KC& k, Ops& o) {
  const bool rho_ok = u[0] > 0.0;
  const double rr = o.rcp(u[0]);
  q[0] = u[0];
  q[1] = o.div(u[1], u[0], rr);
  q[2] = o.div(u[2], u[0], rr);
  q[3] = o.div(u[3], u[0], rr);
  q[4] = u[4];
  q[5] = u[5];
  q[6] = u[6];
  const double m2 = (u[1] * u[1] + u[2] * u[2]) + u[3] * u[3];
  const double b2 = (u[4] * u[4] + u[5] * u[5]) + u[6] * u[6];
  const double internal =
      (u[7] - o.div(0.5 * m2, u[0], rr)) - o.div(b2, k.c.two_mu0, k.r_two_mu0);
  const double p = k.c.gm1 * internal;
  const bool p_ok = p > 0.0;
  const bool floor = !p_ok && k.c.pressure_floor > 0.0;
  q[7] = floor ? k.c.pressure_floor : p;
  if (!rho_ok) return 1;
  return (p_ok || floor) ? 0 : 2;
}

// ppm1d.cpp:14-24 limited_slope with hoisted geometry, branch-free:
//   c0 = dx_k/((dx_{k-1}+dx_k)+dx_{k+1}), A = (2dx_{k-1}+dx_k)/(dx_{k+1}+dx_k),
//   B = (dx_k+2dx_{k+1})/(dx_{k-1}+dx_k)   (bit-exact: same subexpressions).
__device__ __forceinline__ double limited_slope(double qm, double q0, double qp, double c0,
                                                double A, double B) {
  const double dql = q0 - qm;
  const double dqr = qp - q0;
  const double dq = c0 * (A * dqr + B * dql);
  const double lim = 2.0 * smin(fabs(dql), fabs(dqr));
  const double lim_dq = copysign(smin(fabs(dq), lim), dq);
#if defined(PPMLR_FAST_MATH) && PPMLR_FAST_SLOPE_SIGN
  // dqr*dql <= 0 without the FP64 product: opposite sign bits, or a zero
  // difference (then lim = 0 and lim_dq = +-0)
  return ((__double2hiint(dql) ^ __double2hiint(dqr)) < 0) ? 0.0 : lim_dq;
#else
  return (dqr * dql <= 0.0) ? 0.0 : lim_dq;
#endif
}

// Geometry tables per strip position / edge (block.cu build_axis_tables).
// Strict: the reference's own factors (limited_slope c0, A, B; CW84 e0..e4).
// Fast: folded into fewer factors -- slopes (c0 A, c0 B), interface values
// (e0 + e1 e2, -e1 e3, e1 e4) -- fewer FP64 operations and live registers
// per zone, same values to rounding.
#ifdef PPMLR_FAST_MATH
constexpr int kSlopeN = 2, kQfcN = 3;
#else
constexpr int kSlopeN = 3, kQfcN = 5;
#endif
struct SlopeC {
  double c[kSlopeN];
};
__device__ __forceinline__ SlopeC slope_coef(const double* t, int q) {
  SlopeC s;
#pragma unroll
  for (int j = 0; j < kSlopeN; ++j) s.c[j] = __ldg(t + kSlopeN * q + j);
  return s;
}

// ppm1d.cpp:217-224 CW84 interface value at edge m (i = m-1) with hoisted e0..e4.
__device__ __forceinline__ double interface_value(double qi, double qi1, double dmi,
                                                  double dmi1, const double* e) {
  const double dqr = qi1 - qi;
  return (qi + e[0] * dqr) + e[1] * ((e[2] * dqr - e[3] * dmi1) + e[4] * dmi);
}

// The interface value from the block's table entry (strict: e0..e4 in the
// reference's order; fast: the three folded factors).
__device__ __forceinline__ double iface(double qi, double qi1, double dmi, double dmi1,
                                        const double* e) {
#ifdef PPMLR_FAST_MATH
  return (qi + e[0] * (qi1 - qi)) + (e[1] * dmi1 + e[2] * dmi);
#else
  return interface_value(qi, qi1, dmi, dmi1, e);
#endif
}

// limited_slope with the block's table entry for the position.
__device__ __forceinline__ double slope_with(double qm, double q0, double qp, const SlopeC& s) {
#ifdef PPMLR_FAST_MATH
  const double dql = q0 - qm;
  const double dqr = qp - q0;
  const double dq = s.c[0] * dqr + s.c[1] * dql;
  const double lim = 2.0 * smin(fabs(dql), fabs(dqr));
  const double lim_dq = copysign(smin(fabs(dq), lim), dq);
#if PPMLR_FAST_SLOPE_SIGN
  return ((__double2hiint(dql) ^ __double2hiint(dqr)) < 0) ? 0.0 : lim_dq;
#else
  return (dqr * dql <= 0.0) ? 0.0 : lim_dq;
#endif
#else
  return limited_slope(qm, q0, qp, s.c[0], s.c[1], s.c[2]);
#endif
}

// ppm1d.cpp:232-246 monotonicity limiter, branch-free.  ((-d)*d)/6 equals
// -((d*d)/6) exactly, so one quotient serves both comparisons; the steepened
// values use the unmodified al / ar exactly as the reference's if/else chain.
template <class Ops>
__device__ __forceinline__ void limit_parabola(double& al, double& ar, double av, double& six,
                                               const KC& k, Ops& o) {
  const bool flat = (ar - av) * (av - al) <= 0.0;
  const double d = ar - al;
  const double t = d * (av - 0.5 * (al + ar));
  const double x = o.div(d * d, 6.0, k.r6);
  const bool up = t > x;
  const bool dn = !up && t < -x;
  const double al_s = 3.0 * av - 2.0 * ar;
  const double ar_s = 3.0 * av - 2.0 * al;
  al = flat ? av : (up ? al_s : al);
  ar = flat ? av : (dn ? ar_s : ar);
  six = 6.0 * (av - 0.5 * (al + ar));
}

// Fast build: limit_parabola + avg_left/avg_right in one, with the limited
// six and (ar' - al') selected instead of recomputed (algebraically equal:
// up -> six = ar'-al' = 3(ar-av); down -> six = -(ar'-al') = 3(al-av);
// else six = 6(av - (al+ar)/2), ar'-al' = ar-al; flat -> 0), and the
// steepening test t > d^2/6 taken as 2t > d^2/3 on m2 = 2av - (al+ar).
__device__ __forceinline__ void traced_lr(double al, double ar, double av, double hs, double tw,
                                          double r3, double& L, double& R) {
  const double dr = ar - av, dl = av - al;
  const bool flat = dr * dl <= 0.0;
  const double d = ar - al;
  const double m2 = fma(2.0, av, -(al + ar));
  const double t2 = d * m2;
  const double x2 = (d * d) * r3;
  const bool up = t2 > x2;
  const bool dn = !up && t2 < -x2;
  const double av3 = 3.0 * av;
  const double l = flat ? av : (up ? fma(-2.0, ar, av3) : al);
  const double r = flat ? av : (dn ? fma(-2.0, al, av3) : ar);
  const double six = flat ? 0.0 : 3.0 * (up ? dr : (dn ? -dl : m2));
  const double diff = flat ? 0.0 : (up ? six : (dn ? -six : d));
  L = fma(hs, fma(tw, six, diff), l);
  R = fma(-hs, fma(-tw, six, diff), r);
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
template <class Ops>
__device__ __forceinline__ double tw_of(double sigma, const KC& k, Ops& o) {
  return 1.0 - o.div(2.0 * sigma, 3.0, k.r3);
}

// ppm1d.cpp:69-109 solve_edge + edge_flux.  ql/qr strip-frame traced states,
// bl/br total-field offsets (bd components in strip order a, b, d).
template <class QL, class QR, class Ops, bool BD = true>
__device__ __forceinline__ double solve_edge(const QL& ql, const QR& qr,
                                             const double* bl, const double* br, const KC& k,
                                             double* f, Ops& o) {
  const Consts& c = k.c;
  const double wl =
      ql[kRho] * (BD ? fast_speed_strip(ql[kRho], ql[kPE], ql[kBn] + bl[0], ql[kBt1] + bl[1],
                                        ql[kBt2] + bl[2], k, o)
                     : fast_speed_strip(ql[kRho], ql[kPE], ql[kBn], ql[kBt1], ql[kBt2], k, o));
  const double wr =
      qr[kRho] * (BD ? fast_speed_strip(qr[kRho], qr[kPE], qr[kBn] + br[0], qr[kBt1] + br[1],
                                        qr[kBt2] + br[2], k, o)
                     : fast_speed_strip(qr[kRho], qr[kPE], qr[kBn], qr[kBt1], qr[kBt2], k, o));
  const double pl = ql[kPE] + o.div((ql[kBt1] * ql[kBt1] + ql[kBt2] * ql[kBt2]) -
                                        ql[kBn] * ql[kBn],
                                    c.two_mu0, k.r_two_mu0);
  const double pr = qr[kPE] + o.div((qr[kBt1] * qr[kBt1] + qr[kBt2] * qr[kBt2]) -
                                        qr[kBn] * qr[kBn],
                                    c.two_mu0, k.r_two_mu0);
  const double wsum = wl + wr;
  const double r_ws = o.rcp(wsum);
  const double ustar = o.div(((wl * ql[kUn] + wr * qr[kUn]) + pl) - pr, wsum, r_ws);
  const double pstar = o.div((wr * pl + wl * pr) + (wl * wr) * (ql[kUn] - qr[kUn]), wsum, r_ws);
  const double bn = 0.5 * (ql[kBn] + qr[kBn]);
  const double s = bn < 0.0 ? -1.0 : 1.0;
  double al, ar;
  if constexpr (Ops::kFastMath && PPMLR_FAST_RCP_SHARE) {
    al = o.rsq(c.mu0 * ql[kRho]);
    ar = o.rsq(c.mu0 * qr[kRho]);
  } else {
    al = o.dv(1.0, o.sq(c.mu0 * ql[kRho]));
    ar = o.dv(1.0, o.sq(c.mu0 * qr[kRho]));
  }
  const double asum = al + ar;
  const double r_as = o.rcp(asum);
  const double bt1 = o.div((s * (qr[kUt1] - ql[kUt1]) + ar * qr[kBt1]) + al * ql[kBt1], asum, r_as);
  const double bt2 = o.div((s * (qr[kUt2] - ql[kUt2]) + ar * qr[kBt2]) + al * ql[kBt2], asum, r_as);
  const double vt1 = ql[kUt1] + (s * al) * (bt1 - ql[kBt1]);
  const double vt2 = ql[kUt2] + (s * al) * (bt2 - ql[kBt2]);
  f[kRho] = 0.0;
  f[kUn] = pstar;
  f[kUt1] = o.div((-bn) * bt1, c.mu0, k.r_mu0);
  f[kUt2] = o.div((-bn) * bt2, c.mu0, k.r_mu0);
  f[kBn] = (-ustar) * bn;
  f[kBt1] = (-bn) * vt1;
  f[kBt2] = (-bn) * vt2;
  f[kPE] = pstar * ustar - o.div(bn * (vt1 * bt1 + vt2 * bt2), c.mu0, k.r_mu0);
  return ustar;
}

// Runs `body(ops)` with FastOps and, if any fast-path guard failed, again
// with ExactOps (plain `/` and `sqrt`): the item's results are bit-identical
// to the reference in both cases; the second run is rare.
template <class F>
__device__ __forceinline__ void exact_item(F&& body) {
  FastOps fo;
  body(fo);
  if (fo.bad) {
    ExactOps eo;
    body(eo);
  }
}

}  // namespace PPMLR_KNS
}  // namespace ppmlr_b200
