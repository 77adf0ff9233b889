/* ppmlr_oracle.c — plain-C restatement of the reference hot path.
 * TEST INFRASTRUCTURE ONLY; see ppmlr_oracle.h for the contract.
 *
 * Each expression keeps the reference's C++ parse tree (left-to-right for
 * same-precedence operators), so with -ffp-contract=off every rounding step
 * is the reference's.  Citations are to /root/reference/proj.
 */
#include "ppmlr_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

enum { RHO = 0, UN, UT1, UT2, BN, BT1, BT2, PE };

typedef struct {
  double left, right, avg, six;
} parab;

static void set_msg(char* msg, int msglen, const char* s) {
  if (msg && msglen > 0) {
    strncpy(msg, s, (size_t)msglen - 1);
    msg[msglen - 1] = 0;
  }
}

/* std::min / std::max / std::clamp semantics (NaN-order faithful). */
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double sclamp(double v, double lo, double hi) {
  return (v < lo) ? lo : (hi < v) ? hi : v;
}

/* ---- physics (proj/src/physics.cpp) --------------------------------- */

/* physics.cpp:29-37 prim_to_cons; norm2 = (x*x + y*y) + z*z (types.hpp:28-36) */
static void prim_to_cons3(const double* s, double* u, const orc_consts* c) {
  u[0] = s[0];
  u[1] = s[1] * s[0];
  u[2] = s[2] * s[0];
  u[3] = s[3] * s[0];
  u[4] = s[4];
  u[5] = s[5];
  u[6] = s[6];
  const double v2 = (s[1] * s[1] + s[2] * s[2]) + s[3] * s[3];
  const double b2 = (s[4] * s[4] + s[5] * s[5]) + s[6] * s[6];
  u[7] = (s[7] / (c->gamma - 1.0) + (0.5 * s[0]) * v2) + b2 / (2.0 * c->mu0);
}

/* physics.cpp:39-57 cons_to_prim.  Returns 0, or 2 with *bad = offending value
 * and *which = 0 (density) / 1 (pressure). */
static int cons_to_prim3(const double* u, double* q, const orc_consts* c, double* bad,
                         int* which) {
  if (!(u[0] > 0.0)) {
    *bad = u[0];
    *which = 0;
    return 2;
  }
  q[0] = u[0];
  q[1] = u[1] / u[0];
  q[2] = u[2] / u[0];
  q[3] = u[3] / u[0];
  q[4] = u[4];
  q[5] = u[5];
  q[6] = u[6];
  const double m2 = (u[1] * u[1] + u[2] * u[2]) + u[3] * u[3];
  const double b2 = (u[4] * u[4] + u[5] * u[5]) + u[6] * u[6];
  const double internal = (u[7] - (0.5 * m2) / u[0]) - b2 / (2.0 * c->mu0);
  q[7] = (c->gamma - 1.0) * internal;
  if (!(q[7] > 0.0)) {
    if (c->pressure_floor > 0.0) {
      q[7] = c->pressure_floor;
    } else {
      *bad = q[7];
      *which = 1;
      return 2;
    }
  }
  return 0;
}

/* physics.cpp:63-72 fast_speed with total field b = B' + bd (xyz order). */
static double fast_speed3(const double* s, int dir, const orc_consts* c, const double* bd) {
  double b[3];
  for (int i = 0; i < 3; ++i) b[i] = s[4 + i] + (bd ? bd[i] : 0.0);
  const double a2 = (c->gamma * s[7]) / s[0];
  const double ca2 = ((b[0] * b[0] + b[1] * b[1]) + b[2] * b[2]) / (c->mu0 * s[0]);
  const double can2 = (b[dir] * b[dir]) / (c->mu0 * s[0]);
  const double sum = a2 + ca2;
  const double disc = sqrt(smax(0.0, sum * sum - (4.0 * a2) * can2));
  return sqrt(0.5 * (sum + disc));
}

/* ---- 1-D kernel (proj/src/ppm1d.cpp) -------------------------------- */

/* ppm1d.cpp:14-24 */
static double limited_slope(const double* q, const double* dx, int k) {
  const double dql = q[k] - q[k - 1];
  const double dqr = q[k + 1] - q[k];
  if (dqr * dql <= 0.0) return 0.0;
  const double dq =
      (dx[k] / ((dx[k - 1] + dx[k]) + dx[k + 1])) *
      (((2.0 * dx[k - 1] + dx[k]) / (dx[k + 1] + dx[k])) * dqr +
       ((dx[k] + 2.0 * dx[k + 1]) / (dx[k - 1] + dx[k])) * dql);
  const double lim = 2.0 * smin(fabs(dql), fabs(dqr));
  return copysign(smin(fabs(dq), lim), dq);
}

/* ppm1d.cpp:200-247 reconstruct (q, dx length nn; par length nn; work nn+1+nn) */
static void reconstruct(const double* q, const double* dx, int nn, parab* par,
                        double* dm, double* qf) {
  if (nn < 5) {
    for (int i = 0; i < nn; ++i) par[i] = (parab){q[i], q[i], q[i], 0.0};
    return;
  }
  for (int k = 0; k < nn; ++k) dm[k] = 0.0;
  for (int k = 1; k + 1 < nn; ++k) dm[k] = limited_slope(q, dx, k);
  for (int m = 0; m <= nn; ++m) qf[m] = 0.0;
  for (int m = 2; m + 1 < nn; ++m) {
    const int i = m - 1;
    const double dqr = q[i + 1] - q[i];
    const double span = ((dx[i - 1] + dx[i]) + dx[i + 1]) + dx[i + 2];
    const double t1 = ((((2.0 * dx[i + 1]) * dx[i]) / (dx[i] + dx[i + 1])) *
                       ((dx[i - 1] + dx[i]) / (2.0 * dx[i] + dx[i + 1]) -
                        (dx[i + 2] + dx[i + 1]) / (2.0 * dx[i + 1] + dx[i]))) *
                      dqr;
    const double t2 = ((dx[i] * (dx[i - 1] + dx[i])) / (2.0 * dx[i] + dx[i + 1])) * dm[i + 1];
    const double t3 =
        ((dx[i + 1] * (dx[i + 1] + dx[i + 2])) / (dx[i] + 2.0 * dx[i + 1])) * dm[i];
    qf[m] = (q[i] + (dx[i] / (dx[i] + dx[i + 1])) * dqr) + (1.0 / span) * ((t1 - t2) + t3);
  }
  for (int k = 0; k < nn; ++k) {
    if (k < 2 || k >= nn - 2) {
      par[k] = (parab){q[k], q[k], q[k], 0.0};
      continue;
    }
    double al = qf[k], ar = qf[k + 1];
    const double av = q[k];
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
    par[k] = (parab){al, ar, av, 6.0 * (av - 0.5 * (al + ar))};
  }
}

/* ppm1d.hpp:20-26 */
static inline double avg_left(const parab* p, double sigma) {
  return p->left +
         (0.5 * sigma) * ((p->right - p->left) + (1.0 - (2.0 * sigma) / 3.0) * p->six);
}
static inline double avg_right(const parab* p, double sigma) {
  return p->right -
         (0.5 * sigma) * ((p->right - p->left) - (1.0 - (2.0 * sigma) / 3.0) * p->six);
}

/* ppm1d.cpp:29-37 fast_speed_strip (strip-order |B|^2) */
static double fast_speed_strip(double rho, double p, double btn, double btt1, double btt2,
                               const orc_consts* c) {
  const double a2 = (c->gamma * p) / rho;
  const double ca2 = ((btn * btn + btt1 * btt1) + btt2 * btt2) / (c->mu0 * rho);
  const double can2 = (btn * btn) / (c->mu0 * rho);
  const double sum = a2 + ca2;
  const double disc = sqrt(smax(0.0, sum * sum - (4.0 * a2) * can2));
  return sqrt(0.5 * (sum + disc));
}

/* ppm1d.cpp:39-52 prim_to_cons_strip (strip-order sums) */
static void prim_to_cons_strip(const double* w, double* u, const orc_consts* c) {
  u[RHO] = w[RHO];
  u[UN] = w[RHO] * w[UN];
  u[UT1] = w[RHO] * w[UT1];
  u[UT2] = w[RHO] * w[UT2];
  u[BN] = w[BN];
  u[BT1] = w[BT1];
  u[BT2] = w[BT2];
  u[PE] = (w[PE] / (c->gamma - 1.0) +
           (0.5 * w[RHO]) * ((w[UN] * w[UN] + w[UT1] * w[UT1]) + w[UT2] * w[UT2])) +
          ((w[BN] * w[BN] + w[BT1] * w[BT1]) + w[BT2] * w[BT2]) / (2.0 * c->mu0);
}

/* ppm1d.cpp:366-383 strip frame: (a, a+1, a+2 mod 3) */
static void to_strip(const double* s, int dir, double* w) {
  const int a = dir, b = (dir + 1) % 3, d = (dir + 2) % 3;
  w[RHO] = s[0];
  w[UN] = s[1 + a];
  w[UT1] = s[1 + b];
  w[UT2] = s[1 + d];
  w[BN] = s[4 + a];
  w[BT1] = s[4 + b];
  w[BT2] = s[4 + d];
  w[PE] = s[7];
}

/* ppm1d.cpp:69-109 solve_edge + edge_flux; returns u* and writes flux[8]. */
static double solve_edge(const double* ql, const double* qr, const double* bdl,
                         const double* bdr, int dir, const orc_consts* c, double* f) {
  const int a = dir, b = (dir + 1) % 3, d = (dir + 2) % 3;
  const double zl[3] = {0, 0, 0};
  if (!bdl) bdl = zl;
  if (!bdr) bdr = zl;
  const double wl = ql[RHO] * fast_speed_strip(ql[RHO], ql[PE], ql[BN] + bdl[a],
                                               ql[BT1] + bdl[b], ql[BT2] + bdl[d], c);
  const double wr = qr[RHO] * fast_speed_strip(qr[RHO], qr[PE], qr[BN] + bdr[a],
                                               qr[BT1] + bdr[b], qr[BT2] + bdr[d], c);
  const double pl =
      ql[PE] + ((ql[BT1] * ql[BT1] + ql[BT2] * ql[BT2]) - ql[BN] * ql[BN]) / (2.0 * c->mu0);
  const double pr =
      qr[PE] + ((qr[BT1] * qr[BT1] + qr[BT2] * qr[BT2]) - qr[BN] * qr[BN]) / (2.0 * c->mu0);
  const double wsum = wl + wr;
  const double ustar = (((wl * ql[UN] + wr * qr[UN]) + pl) - pr) / wsum;
  const double pstar = ((wr * pl + wl * pr) + (wl * wr) * (ql[UN] - qr[UN])) / wsum;
  const double bn = 0.5 * (ql[BN] + qr[BN]);
  const double s = bn < 0.0 ? -1.0 : 1.0;
  const double al = 1.0 / sqrt(c->mu0 * ql[RHO]);
  const double ar = 1.0 / sqrt(c->mu0 * qr[RHO]);
  const double asum = al + ar;
  const double bt1 = ((s * (qr[UT1] - ql[UT1]) + ar * qr[BT1]) + al * ql[BT1]) / asum;
  const double bt2 = ((s * (qr[UT2] - ql[UT2]) + ar * qr[BT2]) + al * ql[BT2]) / asum;
  const double vt1 = ql[UT1] + (s * al) * (bt1 - ql[BT1]);
  const double vt2 = ql[UT2] + (s * al) * (bt2 - ql[BT2]);
  f[RHO] = 0.0;
  f[UN] = pstar;
  f[UT1] = ((-bn) * bt1) / c->mu0;
  f[UT2] = ((-bn) * bt2) / c->mu0;
  f[BN] = (-ustar) * bn;
  f[BT1] = (-bn) * vt1;
  f[BT2] = (-bn) * vt2;
  f[PE] = pstar * ustar - (bn * (vt1 * bt1 + vt2 * bt2)) / c->mu0;
  return ustar;
}

/* ppm1d.cpp:111-196 lagrangian_phase + 317-364 sweep_1d */
int orc_sweep_1d(double* states, const double* bd, const double* dx, int n, int ghost,
                 double dt, int dir, const orc_consts* c, char* msg, int msglen) {
  const int nn = n + 2 * ghost;
  double* prim = malloc(sizeof(double) * 8 * nn);
  double* cons = malloc(sizeof(double) * 8 * nn);
  double* cf = malloc(sizeof(double) * nn);
  parab* ppar = malloc(sizeof(parab) * 8 * nn);
  parab* cpar = malloc(sizeof(parab) * 8 * nn);
  double* scratch = malloc(sizeof(double) * nn);
  double* dm = malloc(sizeof(double) * nn);
  double* qf = malloc(sizeof(double) * (nn + 1));
  double* flux = calloc((size_t)8 * (nn + 1), sizeof(double));
  double* uedge = calloc((size_t)(nn + 1), sizeof(double));
  double* lag = calloc((size_t)8 * nn, sizeof(double));
  double* widths = calloc((size_t)nn, sizeof(double));
  int rc = 0;
  char buf[256];

  for (int i = 0; i < nn; ++i) {
    to_strip(states + 8 * i, dir, prim + 8 * i);
    prim_to_cons_strip(prim + 8 * i, cons + 8 * i, c);
    cf[i] = fast_speed3(states + 8 * i, dir, c, bd ? bd + 3 * i : NULL);
  }
  for (int v = 0; v < 8; ++v) {
    for (int i = 0; i < nn; ++i) scratch[i] = prim[8 * i + v];
    reconstruct(scratch, dx, nn, ppar + (size_t)v * nn, dm, qf);
    for (int i = 0; i < nn; ++i) scratch[i] = cons[8 * i + v];
    reconstruct(scratch, dx, nn, cpar + (size_t)v * nn, dm, qf);
  }

  /* traced states, ppm1d.cpp:136-145 */
  const int first_edge = 3, last_edge = nn - 2;
  for (int m = first_edge; m <= last_edge; ++m) {
    double ql[8], qr[8];
    for (int side = 0; side < 2; ++side) {
      const int zone = side == 0 ? m - 1 : m;
      double* q = side == 0 ? ql : qr;
      const double sigma = sclamp((cf[zone] * dt) / dx[zone], 0.0, 1.0);
      for (int v = 0; v < 8; ++v)
        q[v] = side == 0 ? avg_right(&ppar[(size_t)v * nn + zone], sigma)
                         : avg_left(&ppar[(size_t)v * nn + zone], sigma);
      if (!(q[RHO] > 0.0) || !(q[PE] > 0.0))
        for (int v = 0; v < 8; ++v) q[v] = prim[8 * zone + v];
    }
    uedge[m] = solve_edge(ql, qr, bd ? bd + 3 * (m - 1) : NULL, bd ? bd + 3 * m : NULL, dir,
                          c, flux + 8 * m);
  }

  /* Lagrangian update, ppm1d.cpp:175-194 */
  for (int k = first_edge; k <= last_edge - 1; ++k) {
    const double dx0 = dx[k];
    const double dxp = dx0 + dt * (uedge[k + 1] - uedge[k]);
    if (!(dxp > 0.0)) {
      snprintf(buf, sizeof buf, "Lagrangian interfaces crossed at zone %d", k);
      set_msg(msg, msglen, buf);
      rc = 3;
      goto done;
    }
    const double shrink = dx0 / dxp;
    for (int v = 0; v < 8; ++v)
      lag[8 * k + v] =
          cons[8 * k + v] * shrink - (dt * (flux[8 * (k + 1) + v] - flux[8 * k + v])) / dxp;
    widths[k] = dxp;
    if (c->pressure_floor <= 0.0) {
      const double* u = lag + 8 * k;
      const double internal =
          (u[PE] - (0.5 * ((u[UN] * u[UN] + u[UT1] * u[UT1]) + u[UT2] * u[UT2])) / u[RHO]) -
          ((u[BN] * u[BN] + u[BT1] * u[BT1]) + u[BT2] * u[BT2]) / (2.0 * c->mu0);
      if (!(u[RHO] > 0.0) || !(internal > 0.0)) {
        snprintf(buf, sizeof buf,
                 "negative density or pressure after Lagrangian step at zone %d", k);
        set_msg(msg, msglen, buf);
        rc = 2;
        goto done;
      }
    }
  }

  /* remap with carried parabolas, ppm1d.cpp:325-361 */
  {
    const int a = dir, b = (dir + 1) % 3, d = (dir + 2) % 3;
    for (int j = ghost; j < ghost + n; ++j) {
      const double dxe = dx[j];
      const double scale = widths[j] / dxe;
      double u[8];
      for (int v = 0; v < 8; ++v) {
        double sl[2];
        for (int e = 0; e < 2; ++e) {
          const int m = j + e;
          const double delta = uedge[m] * dt;
          if (delta == 0.0) {
            sl[e] = 0.0;
          } else if (delta > 0.0) {
            const int k = m - 1;
            const double carried = avg_right(&cpar[(size_t)v * nn + k], delta / widths[k]) +
                                   (lag[8 * k + v] - cons[8 * k + v]);
            sl[e] = delta * carried;
          } else {
            const int k = m;
            const double carried =
                avg_left(&cpar[(size_t)v * nn + k], (-delta) / widths[k]) +
                (lag[8 * k + v] - cons[8 * k + v]);
            sl[e] = delta * carried;
          }
        }
        u[v] = lag[8 * j + v] * scale + (sl[0] - sl[1]) / dxe;
      }
      double cs[8], q[8], bad;
      int which;
      cs[0] = u[RHO];
      cs[1 + a] = u[UN];
      cs[1 + b] = u[UT1];
      cs[1 + d] = u[UT2];
      cs[4 + a] = u[BN];
      cs[4 + b] = u[BT1];
      cs[4 + d] = u[BT2];
      cs[7] = u[PE];
      if (cons_to_prim3(cs, q, c, &bad, &which)) {
        if (which == 0)
          snprintf(buf, sizeof buf, "non-positive density %f at strip cell %d", bad, j - ghost);
        else
          snprintf(buf, sizeof buf,
                   "non-positive pressure %f recovered from conserved state at strip cell %d",
                   bad, j - ghost);
        set_msg(msg, msglen, buf);
        rc = 2;
        goto done;
      }
      memcpy(states + 8 * j, q, sizeof q);
    }
  }
done:
  free(prim);
  free(cons);
  free(cf);
  free(ppar);
  free(cpar);
  free(scratch);
  free(dm);
  free(qf);
  free(flux);
  free(uedge);
  free(lag);
  free(widths);
  return rc;
}

double orc_strip_max_dt(const double* states, const double* bd, const double* dx, int n,
                        int ghost, int dir, const orc_consts* c) {
  double dt = INFINITY;
  for (int i = ghost; i < ghost + n; ++i) {
    const double cf = fast_speed3(states + 8 * i, dir, c, bd ? bd + 3 * i : NULL);
    const double speed = fabs(states[8 * i + 1 + dir]) + cf;
    dt = smin(dt, dx[i] / speed);
  }
  return dt;
}

/* ---- 3-D block stepper (proj/src/stepper.cpp) ----------------------- */

static inline int64_t span_of(const orc_block* b, int a) { return b->n[a] + 2 * b->ghost; }
static inline int64_t idx_of(const orc_block* b, int i, int j, int k) {
  const int g = b->ghost;
  return (int64_t)(i + g) + span_of(b, 0) * ((int64_t)(j + g) + span_of(b, 1) * (k + g));
}

/* stepper.cpp:119-139 */
int orc_compute_dt(const orc_block* b, double cfl, const orc_consts* c, double* dt_out,
                   char* msg, int msglen) {
  double dt = INFINITY;
  for (int k = 0; k < b->n[2]; ++k)
    for (int j = 0; j < b->n[1]; ++j)
      for (int i = 0; i < b->n[0]; ++i) {
        const int64_t idx = idx_of(b, i, j, k);
        const double* s = b->fields + 8 * idx;
        const int local[3] = {i + b->ghost, j + b->ghost, k + b->ghost};
        for (int a = 0; a < 3; ++a) {
          const double cf = fast_speed3(s, a, c, b->bd ? b->bd + 3 * idx : NULL);
          const double speed = fabs(s[1 + a]) + cf;
          const double cand = b->spacings[a][local[a]] / speed;
          if (!isfinite(cand)) {
            char buf[128];
            snprintf(buf, sizeof buf, "non-finite signal speed at cell (%d,%d,%d)", i, j, k);
            set_msg(msg, msglen, buf);
            return 2;
          }
          dt = smin(dt, cand);
        }
      }
  *dt_out = cfl * dt;
  return 0;
}

/* stepper.cpp:42-45 */
static inline double central_diff(double fm, double f0, double fp, double hm, double hp) {
  return (((hm * hm) * fp + ((hp * hp) - (hm * hm)) * f0) - (hp * hp) * fm) /
         ((hm * hp) * (hm + hp));
}

static inline void cross3(const double* a, const double* b, double* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

/* stepper.cpp:141-200 */
int orc_apply_sources(orc_block* b, double dt, const orc_consts* c, char* msg, int msglen) {
  const int g = b->ghost;
  const int64_t cells = span_of(b, 0) * span_of(b, 1) * span_of(b, 2);
  double* updated = malloc(sizeof(double) * 8 * (size_t)cells);
  static const double zero3[3] = {0, 0, 0};
  for (int k = 0; k < b->n[2]; ++k)
    for (int j = 0; j < b->n[1]; ++j)
      for (int i = 0; i < b->n[0]; ++i) {
        const int64_t idx = idx_of(b, i, j, k);
        const double* s = b->fields + 8 * idx;
        const double* bd0 = b->bd ? b->bd + 3 * idx : zero3;
        double grad_b[3][3], grad_e[3][3];
        for (int a = 0; a < 3; ++a) {
          int im[3] = {i, j, k}, ip[3] = {i, j, k};
          im[a] -= 1;
          ip[a] += 1;
          const int64_t idm = idx_of(b, im[0], im[1], im[2]);
          const int64_t idp = idx_of(b, ip[0], ip[1], ip[2]);
          const int lc = (a == 0 ? i : (a == 1 ? j : k)) + g;
          const double hm = b->centers[a][lc] - b->centers[a][lc - 1];
          const double hp = b->centers[a][lc + 1] - b->centers[a][lc];
          const double* sm = b->fields + 8 * idm;
          const double* sp = b->fields + 8 * idp;
          double em[3], e0[3], ep[3];
          cross3(sm + 1, b->bd ? b->bd + 3 * idm : zero3, em);
          cross3(s + 1, bd0, e0);
          cross3(sp + 1, b->bd ? b->bd + 3 * idp : zero3, ep);
          for (int comp = 0; comp < 3; ++comp) {
            grad_b[a][comp] = central_diff(sm[4 + comp], s[4 + comp], sp[4 + comp], hm, hp);
            grad_e[a][comp] = central_diff(em[comp], e0[comp], ep[comp], hm, hp);
          }
        }
        const double curl_b[3] = {grad_b[1][2] - grad_b[2][1], grad_b[2][0] - grad_b[0][2],
                                  grad_b[0][1] - grad_b[1][0]};
        const double curl_e[3] = {grad_e[1][2] - grad_e[2][1], grad_e[2][0] - grad_e[0][2],
                                  grad_e[0][1] - grad_e[1][0]};
        const double div_b = (grad_b[0][0] + grad_b[1][1]) + grad_b[2][2];
        double s_mom[3];
        cross3(curl_b, bd0, s_mom);
        for (int q = 0; q < 3; ++q) s_mom[q] = s_mom[q] / c->mu0;
        double s_ind[3];
        for (int q = 0; q < 3; ++q) s_ind[q] = curl_e[q] - s[1 + q] * div_b;
        const double s_energy =
            ((s[1] * s_mom[0] + s[2] * s_mom[1]) + s[3] * s_mom[2]) +
            ((s[4] * curl_e[0] + s[5] * curl_e[1]) + s[6] * curl_e[2]) / c->mu0;
        double* u = updated + 8 * idx;
        prim_to_cons3(s, u, c);
        for (int q = 0; q < 3; ++q) u[1 + q] += s_mom[q] * dt;
        for (int q = 0; q < 3; ++q) u[4 + q] += s_ind[q] * dt;
        u[7] += dt * s_energy;
      }
  int rc = 0;
  for (int k = 0; k < b->n[2] && !rc; ++k)
    for (int j = 0; j < b->n[1] && !rc; ++j)
      for (int i = 0; i < b->n[0]; ++i) {
        const int64_t idx = idx_of(b, i, j, k);
        double q[8], bad;
        int which;
        if (cons_to_prim3(updated + 8 * idx, q, c, &bad, &which)) {
          char buf[256];
          if (which == 0)
            snprintf(buf, sizeof buf, "non-positive density %f after sources at cell (%d,%d,%d)",
                     bad, i, j, k);
          else
            snprintf(buf, sizeof buf,
                     "non-positive pressure %f recovered from conserved state after sources "
                     "at cell (%d,%d,%d)",
                     bad, i, j, k);
          set_msg(msg, msglen, buf);
          rc = 2;
          break;
        }
        memcpy(b->fields + 8 * idx, q, sizeof q);
      }
  free(updated);
  return rc;
}

/* stepper.cpp:202-247 */
int orc_apply_boundaries(orc_block* b, const orc_opts* o, char* msg, int msglen) {
  const int g = b->ghost;
  for (int a = 0; a < 3; ++a) {
    if (o->boundary == 1) {
      if (b->physical[a][0] != b->physical[a][1] || (b->physical[a][0] && b->n[a] < g)) {
        set_msg(msg, msglen, "periodic boundaries need whole-axis blocks");
        return 1;
      }
    }
    for (int side = 0; side < 2; ++side) {
      if (!b->physical[a][side]) continue;
      const int nb = b->n[(a + 1) % 3], nc = b->n[(a + 2) % 3];
      for (int t2 = 0; t2 < nc; ++t2)
        for (int t1 = 0; t1 < nb; ++t1)
          for (int layer = 1; layer <= g; ++layer) {
            int cell[3], src[3];
            cell[(a + 1) % 3] = src[(a + 1) % 3] = t1;
            cell[(a + 2) % 3] = src[(a + 2) % 3] = t2;
            cell[a] = side == 0 ? -layer : b->n[a] - 1 + layer;
            double* dst = b->fields + 8 * idx_of(b, cell[0], cell[1], cell[2]);
            if (o->boundary == 1) {
              src[a] = side == 0 ? b->n[a] - layer : layer - 1;
            } else if (o->boundary == 2 && a == 0 && side == 1) {
              const int64_t id = idx_of(b, cell[0], cell[1], cell[2]);
              dst[0] = o->wind_rho;
              dst[7] = o->wind_p;
              for (int q = 0; q < 3; ++q) {
                dst[1 + q] = o->wind_v[q];
                dst[4 + q] = o->wind_imf[q] - (b->bd ? b->bd[3 * id + q] : 0.0);
              }
              continue;
            } else {
              src[a] = side == 0 ? 0 : b->n[a] - 1;
            }
            memcpy(dst, b->fields + 8 * idx_of(b, src[0], src[1], src[2]), 8 * sizeof(double));
          }
    }
  }
  return 0;
}

/* stepper.cpp:249-282 */
int orc_sweep_axis(orc_block* b, int axis, double dt, const orc_consts* c, char* msg,
                   int msglen) {
  const int g = b->ghost;
  const int bb = (axis + 1) % 3, d = (axis + 2) % 3;
  const int n = b->n[axis];
  const int nn = n + 2 * g;
  double* st = malloc(sizeof(double) * 8 * nn);
  double* bdv = b->bd ? malloc(sizeof(double) * 3 * nn) : NULL;
  int rc = 0;
  for (int t2 = 0; t2 < b->n[d] && !rc; ++t2)
    for (int t1 = 0; t1 < b->n[bb]; ++t1) {
      int cell[3];
      cell[bb] = t1;
      cell[d] = t2;
      for (int i = -g; i < n + g; ++i) {
        cell[axis] = i;
        const int64_t idx = idx_of(b, cell[0], cell[1], cell[2]);
        memcpy(st + 8 * (i + g), b->fields + 8 * idx, 8 * sizeof(double));
        if (bdv) memcpy(bdv + 3 * (i + g), b->bd + 3 * idx, 3 * sizeof(double));
      }
      char inner[256];
      const int r = orc_sweep_1d(st, bdv, b->spacings[axis], n, g, dt, axis, c, inner,
                                 sizeof inner);
      if (r) {
        char buf[400];
        snprintf(buf, sizeof buf, "%s in sweep axis %d at line (%d,%d)", inner, axis, t1, t2);
        set_msg(msg, msglen, buf);
        rc = 2; /* stepper.cpp:272-276 rethrows every Error as UnphysicalState */
        break;
      }
      for (int i = 0; i < n; ++i) {
        cell[axis] = i;
        memcpy(b->fields + 8 * idx_of(b, cell[0], cell[1], cell[2]), st + 8 * (i + g),
               8 * sizeof(double));
      }
    }
  free(st);
  free(bdv);
  return rc;
}

void orc_restore_frozen(orc_block* b) {
  for (int64_t f = 0; f < b->n_frozen; ++f)
    memcpy(b->fields + 8 * b->frozen_idx[f], b->frozen_states + 8 * f, 8 * sizeof(double));
}

/* harness.cpp:59-92 with a single (1,1,1) block: exchanges are empty. */
int orc_advance(orc_block* b, const orc_opts* o, const orc_consts* c, long step,
                double* dt_out, char* msg, int msglen) {
  double dt;
  int rc = orc_compute_dt(b, o->cfl, c, &dt, msg, msglen);
  if (rc) return rc;
  const int order[2][3] = {{0, 1, 2}, {2, 1, 0}};
  for (int s = 0; s < 3; ++s) {
    const int axis = order[step % 2 == 0 ? 0 : 1][s];
    rc = orc_apply_boundaries(b, o, msg, msglen);
    if (rc) return rc;
    rc = orc_sweep_axis(b, axis, dt, c, msg, msglen);
    if (rc) return rc;
  }
  if (o->with_sources) {
    rc = orc_apply_boundaries(b, o, msg, msglen);
    if (rc) return rc;
    rc = orc_apply_sources(b, dt, c, msg, msglen);
    if (rc) return rc;
  }
  orc_restore_frozen(b);
  *dt_out = dt;
  return 0;
}
