/* C-ABI shim over the UNMODIFIED reference C++ sources (/root/reference/proj).
 *
 * TEST INFRASTRUCTURE ONLY.  This header and ref_shim.cpp are compiled together
 * with the reference's own src/*.cpp by oracle/Makefile into
 * oracle/_ref/libppmlr_ref.so.  Only tests/, __graft_entry__.smoke() and
 * bench.py's CPU-baseline / --impl reference legs may load it.  The product
 * (paper_1607_02214_b200/) never links or calls it.
 *
 * Every entry point forwards to the reference API it names:
 *   ref_build_axis          -> ppmlr::build_axis        (proj/src/grid.cpp:61-135)
 *   ref_sweep_1d            -> ppmlr::sweep_1d          (proj/src/ppm1d.cpp:317-364)
 *   ref_strip_max_dt        -> ppmlr::strip_max_dt      (proj/src/ppm1d.cpp:307-315)
 *   ref_harness_*           -> ppmlr::Harness           (proj/include/ppmlr/harness.hpp:48-87)
 *   ref_layout              -> ppmlr::layout            (proj/src/decomp.cpp:46-86)
 */
#ifndef PPMLR_REF_SHIM_H
#define PPMLR_REF_SHIM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double min, max, uniform_lo, uniform_hi, d_uniform;
  int cells;
  double ratio;
} ref_axis_spec;

typedef struct {
  double cfl;
  int ghost;
  int boundary;   /* 0 outflow, 1 periodic, 2 magnetosphere */
  int transport;  /* 0 staged, 1 direct */
  int with_sources, with_dipole;
  double wind_rho, wind_p, wind_v[3], wind_imf[3];
  double mu0, gamma, pressure_floor;
} ref_options;

/* Return codes: 0 ok, 1 InvalidSpec, 2 UnphysicalState, 3 StepRejected,
 * 4 OutOfRange, 5 other ppmlr::Error, 6 other std::exception. */

int ref_build_axis(const ref_axis_spec* spec, double* edges, double* centers,
                   double* spacings, int cap, int* n_out, char* err, int errlen);

int ref_sweep_1d(double* states, const double* bd, const double* spacings, int n,
                 int ghost, double dt, int dir, double gamma, double mu0,
                 double pressure_floor, char* err, int errlen);

double ref_strip_max_dt(const double* states, const double* bd, const double* spacings,
                        int n, int ghost, int dir, double gamma, double mu0);

/* layout(): blocks[r*16 + ...] = rank, coords[3], lo[3], n[3], neighbor[6] */
int ref_layout(const ref_axis_spec* specs3, int px, int py, int pz, int* blocks,
               int cap_blocks, int* nblocks, int* iono_rank, char* err, int errlen);

void* ref_harness_create(const ref_axis_spec* specs3, int px, int py, int pz,
                         const ref_options* opts, char* err, int errlen);
void ref_harness_destroy(void* h);
int ref_harness_block_count(void* h);
/* n[3], lo[3], ghost for block r */
void ref_harness_block_dims(void* h, int r, int* n, int* lo, int* ghost);
/* ghost-inclusive geometry of block r along axis a (span doubles each) */
void ref_harness_block_axis(void* h, int r, int a, double* centers, double* spacings);
/* ghost-inclusive AoS fields (8 per cell, BlockState::index order) */
void ref_harness_get_fields(void* h, int r, double* out);
void ref_harness_set_fields(void* h, int r, const double* in);
void ref_harness_get_bd(void* h, int r, double* out);
int64_t ref_harness_frozen_count(void* h, int r);
void ref_harness_get_frozen(void* h, int r, int64_t* idx, double* states);
int ref_harness_init_magnetosphere(void* h, double rho_core, double p_core,
                                   double falloff, double r_ref, char* err, int errlen);
/* Pointwise ICs evaluated at every cell incl. ghosts (Harness::init_with).
 * kind: 0 uniform(params[0..7] = rho,vx,vy,vz,bx,by,bz,p), 1 Brio-Wu,
 * 2 Orszag-Tang(params[0]=gamma), 3 blast per unit block (params: p_in, p_out,
 * radius), 4 verify.cpp partition_ic, 5 acceptance smooth_ic,
 * 6 verify.cpp conservation gaussian. */
int ref_harness_init_ic(void* h, int kind, const double* params, char* err, int errlen);
int ref_harness_advance(void* h, double* dt_out, char* err, int errlen);
int ref_harness_compute_dt(void* h, double* dt_out, char* err, int errlen);
void ref_harness_gather(void* h, double* out);
long ref_harness_step(void* h);
double ref_harness_time(void* h);
uint64_t ref_harness_ledger_bytes(void* h);
long ref_harness_ledger_messages(void* h);
long ref_harness_ledger_copy_events(void* h);
long ref_harness_ledger_entries(void* h, long* step, int* transport, long* messages,
                                uint64_t* bytes, long* copy_events, long max);
/* run_suite (verify.cpp:234-243): count of checks (or -rc on error). */
int ref_run_suite(const char* name, double* metrics, int* pass, int max, char* err,
                  int errlen);
int ref_harness_write_snapshot(void* h, const char* path, char* err, int errlen);

/* CPU baseline: `threads` independent harnesses (one per thread) built from
 * the same spec and IC, each advanced `steps` times.  Returns aggregate
 * cell-updates/s in *rate and the max per-thread wall seconds in *seconds.
 * ic_kind < 0 means init_magnetosphere with default profiles. */
int ref_bench(const ref_axis_spec* specs3, const ref_options* opts, int ic_kind,
              const double* ic_params, int threads, int steps, double* rate,
              double* seconds, char* err, int errlen);

#ifdef __cplusplus
}
#endif
#endif
