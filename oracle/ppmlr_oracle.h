/* ppmlr_oracle — plain-C restatement of the reference PPMLR-MHD hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the CPU checker for the B200 product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load oracle/liboracle.so.  The product never links it and has no CPU
 * fallback.
 *
 * Parity pin: every function restates the reference function cited next to
 * it with the same IEEE-754 binary64 operation order (C left-to-right
 * association, no FMA contraction: built with -ffp-contract=off).  The
 * restatement is checked bit-for-bit against the reference itself
 * (oracle/_ref/libppmlr_ref.so, compiled from /root/reference sources by
 * oracle/Makefile) and against committed golden vectors generated from that
 * build (tests/golden/).
 *
 * Layout conventions are the reference's: a block's state is AoS, 8 doubles
 * per cell (rho, vx, vy, vz, B'x, B'y, B'z, p), linear index
 * (i+g) + S0*((j+g) + S1*(k+g)) with S_a = n_a + 2g
 * (proj/include/ppmlr/stepper.hpp:46-49).
 *
 * Return codes: 0 ok, 1 InvalidSpec, 2 UnphysicalState, 3 StepRejected.
 */
#ifndef PPMLR_ORACLE_H
#define PPMLR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double gamma, mu0, pressure_floor;
} orc_consts;

typedef struct {
  int n[3];
  int ghost;
  const double* centers[3];  /* ghost-inclusive, n[a]+2g each */
  const double* spacings[3]; /* ghost-inclusive */
  int physical[3][2];
  double* fields;            /* AoS, 8 per cell */
  const double* bd;          /* AoS, 3 per cell, or NULL (no dipole) */
  const int64_t* frozen_idx; /* linear indices of the frozen inner core */
  const double* frozen_states; /* 8 per frozen cell */
  int64_t n_frozen;
} orc_block;

typedef struct {
  int boundary; /* 0 outflow, 1 periodic, 2 magnetosphere */
  double wind_rho, wind_p, wind_v[3], wind_imf[3];
  double cfl;
  int with_sources;
} orc_opts;

/* proj/src/ppm1d.cpp:317-364 sweep_1d on one strip: states AoS (n+2g)*8,
 * bd AoS (n+2g)*3 or NULL, dx (n+2g). */
int orc_sweep_1d(double* states, const double* bd, const double* dx, int n, int ghost,
                 double dt, int dir, const orc_consts* c, char* msg, int msglen);
/* proj/src/ppm1d.cpp:307-315 */
double orc_strip_max_dt(const double* states, const double* bd, const double* dx, int n,
                        int ghost, int dir, const orc_consts* c);
/* proj/src/stepper.cpp:119-139 */
int orc_compute_dt(const orc_block* b, double cfl, const orc_consts* c, double* dt,
                   char* msg, int msglen);
/* proj/src/stepper.cpp:202-247 */
int orc_apply_boundaries(orc_block* b, const orc_opts* o, char* msg, int msglen);
/* proj/src/stepper.cpp:249-282 */
int orc_sweep_axis(orc_block* b, int axis, double dt, const orc_consts* c, char* msg,
                   int msglen);
/* proj/src/stepper.cpp:141-200 */
int orc_apply_sources(orc_block* b, double dt, const orc_consts* c, char* msg, int msglen);
/* proj/src/stepper.cpp:284-286 */
void orc_restore_frozen(orc_block* b);
/* Harness::advance for a single whole-domain block, proj/src/harness.cpp:59-92
 * (global dt, XYZ/ZYX sweeps with boundary fills, sources, frozen core). */
int orc_advance(orc_block* b, const orc_opts* o, const orc_consts* c, long step,
                double* dt_out, char* msg, int msglen);

#ifdef __cplusplus
}
#endif
#endif
