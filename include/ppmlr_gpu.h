/* ppmlr_gpu.h — C-ABI of the B200-native PPMLR-MHD time-step hot path.
 *
 * The reference (arxiv 1607.02214, /root/reference/proj) has no plugin or
 * FFI layer: its boundary is the C++ API one level above the numerics
 * (SURVEY.md §8(b)).  This header is the drop-in boundary a C++ (or any FFI)
 * caller binds; every entry point names the reference interface it
 * replaces.  Plain pointers and sizes only; no exceptions cross it.
 *
 * Status codes (ppmlr::Error subclasses, proj/include/ppmlr/errors.hpp:9-30):
 *   0 ok, 1 InvalidSpec, 2 UnphysicalState, 3 StepRejected, 4 OutOfRange,
 *   5 CUDA / runtime failure.
 * The message of the last failure is available from ppmlr_gpu_last_error().
 *
 * State layout at the boundary is the reference's: AoS, 8 doubles per cell
 * (rho, vx, vy, vz, B'x, B'y, B'z, p), ghost-inclusive linear index
 * (i+g) + S0*((j+g) + S1*(k+g)), S_a = n_a + 2g  (stepper.hpp:46-49).
 * On the device the state is structure-of-arrays with a padded x pitch.
 *
 * Ownership: handles own all device memory; caller buffers are borrowed for
 * the duration of a call.  One host thread drives a handle.
 */
#ifndef PPMLR_GPU_H
#define PPMLR_GPU_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { PPMLR_OK = 0, PPMLR_INVALID_SPEC = 1, PPMLR_UNPHYSICAL = 2, PPMLR_STEP_REJECTED = 3,
       PPMLR_OUT_OF_RANGE = 4, PPMLR_RUNTIME = 5 };
/* BoundaryMode, stepper.hpp:29 */
enum { PPMLR_BC_OUTFLOW = 0, PPMLR_BC_PERIODIC = 1, PPMLR_BC_MAGNETOSPHERE = 2 };
/* Arithmetic mode: STRICT is bit-identical to the reference CPU build;
 * FAST contracts FMAs and folds divisions (tolerance-gated). */
enum { PPMLR_STRICT = 0, PPMLR_FAST = 1 };

/* Last error message of the calling thread (any handle or free function). */
const char* ppmlr_gpu_last_error(void);
/* Library version / build string (for provenance in benchmarks). */
const char* ppmlr_gpu_version(void);

/* ------------------------------------------------------------------------
 * Geometry and decomposition (host-side planning code, rewritten natively;
 * results are bit-identical to the reference's).
 * ---------------------------------------------------------------------- */
typedef struct {
  double min, max, uniform_lo, uniform_hi, d_uniform;
  int cells;
  double ratio;
} ppmlr_axis_spec; /* AxisSpec, grid.hpp:9-17 */

/* build_axis (grid.cpp:61-135).  edges cap+1, centers/spacings cap. */
int ppmlr_build_axis(const ppmlr_axis_spec* spec, double* edges, double* centers,
                     double* spacings, int cap, int* n_out);

/* layout (decomp.cpp:46-86).  Per block 16 ints: rank, coords[3], lo[3], n[3],
 * neighbor[6] (-x,+x,-y,+y,-z,+z; -1 = physical face).  violations (if not
 * NULL) receives the validate() messages joined as the reference does. */
int ppmlr_layout(const ppmlr_axis_spec specs[3], int px, int py, int pz, int* blocks,
                 int cap_blocks, int* nblocks, int* ionosphere_rank);
/* tde_units / exchanged_bytes (decomp.cpp:88-108). */
long ppmlr_tde_units(int px, int py, int pz);
uint64_t ppmlr_exchanged_bytes(const ppmlr_axis_spec specs[3], int px, int py, int pz,
                               int ghost, int bytes_per_cell);

/* Host-only (no GPU): the ghost-inclusive initial state, dipole field,
 * frozen core and geometry of block `rank` exactly as the Harness uploads
 * them (make_block stepper.cpp:49-71, init_magnetosphere :83-112 when
 * ic_kind < 0 with params = rho_core, p_core, falloff, r_ref; otherwise
 * init_with of the built-in IC `ic_kind`, harness.cpp:35-43).  Any output
 * pointer may be NULL. */
typedef struct ppmlr_gpu_options ppmlr_gpu_options;
int ppmlr_host_block_state(const ppmlr_axis_spec specs[3], int px, int py, int pz,
                           const ppmlr_gpu_options* opts, int rank, int ic_kind,
                           const double* params, double* fields, double* bd,
                           int64_t* frozen_idx, double* frozen_states, int64_t* n_frozen,
                           double* centers_cat, double* spacings_cat);

/* Number of visible CUDA devices (0 when none / no driver). */
int ppmlr_gpu_device_count(void);
/* Measured FP64 FMA throughput of `device` in TFLOP/s (DFMA-chain
 * microbenchmark; the FP64 roofline denominator). */
int ppmlr_gpu_fp64_peak(int device, double* tflops);
/* Self-test of the bit-exact shared-reciprocal division used by the strict
 * kernels against the compiler's `/` on n generated operand pairs; returns
 * the mismatch count and the first mismatch (a, b, a/b, ours). */
int ppmlr_gpu_selftest_division(int device, long long n, unsigned long long seed,
                                long long* mismatches, double* example4);

/* ------------------------------------------------------------------------
 * Block: one BlockState resident on one GPU (stepper.hpp:33-55) and the
 * per-block operations of Harness::advance (harness.cpp:59-92).
 * ---------------------------------------------------------------------- */
typedef struct ppmlr_gpu_block ppmlr_gpu_block;

typedef struct {
  int n[3];                  /* interior cells per axis */
  int lo[3];                 /* global index of the first interior cell */
  int ghost;                 /* ghost width of the caller's arrays (>= 4) */
  const double* centers[3];  /* ghost-inclusive, n[a] + 2*ghost each */
  const double* spacings[3]; /* ghost-inclusive */
  int physical[3][2];        /* face at the domain boundary */
  double gamma, mu0, pressure_floor;
  int boundary;              /* PPMLR_BC_* */
  double wind_rho, wind_p, wind_v[3], wind_imf[3];
  int with_dipole;           /* bd arrays are uploaded and used */
  int precision;             /* PPMLR_STRICT / PPMLR_FAST */
  int device;                /* CUDA ordinal */
} ppmlr_gpu_block_desc;

/* make_block (stepper.cpp:49-71): allocates the device state. */
int ppmlr_gpu_block_create(const ppmlr_gpu_block_desc* desc, ppmlr_gpu_block** out);
void ppmlr_gpu_block_destroy(ppmlr_gpu_block* b);

/* Host -> device: ghost-inclusive AoS fields, bd (3 per cell, or NULL) and
 * the frozen inner core (init_magnetosphere, stepper.cpp:83-112): linear
 * reference indices + 8 doubles each.  Resets the block's step counter. */
int ppmlr_gpu_block_upload(ppmlr_gpu_block* b, const double* fields, const double* bd,
                           const int64_t* frozen_idx, const double* frozen_states,
                           int64_t n_frozen);
/* Device -> host: ghost-inclusive AoS (ghost shells hold whatever the last
 * fill left; interiors are exact). */
int ppmlr_gpu_block_download(ppmlr_gpu_block* b, double* fields);
/* Device -> host: interior only, AoS x fastest (gather_interior order). */
int ppmlr_gpu_block_download_interior(ppmlr_gpu_block* b, double* out);
/* Snapshot of the current state (the device half of gather_interior ->
 * write_snapshot, tools/ppmlr_main.cpp:20-31, src/snapshot.cpp:58-85):
 * capture copies the interior, field-major and x fastest, to a device
 * buffer in stream order and returns at once; read drains interior planes
 * [k0, k0+nk) of one field (0..7 = rho, vx, vy, vz, B'x, B'y, B'z, p) to
 * host memory on the block's snapshot stream, row pitch / plane slice in
 * doubles, so a caller can place the block inside a global array. */
int ppmlr_gpu_block_snapshot_capture(ppmlr_gpu_block* b);
int ppmlr_gpu_block_snapshot_read(ppmlr_gpu_block* b, int field, int k0, int nk, double* dst,
                                  int64_t dst_pitch, int64_t dst_slice);

/* compute_dt (stepper.cpp:119-139): cfl * min over the block. */
int ppmlr_gpu_block_compute_dt(ppmlr_gpu_block* b, double cfl, double* dt_out);
/* apply_boundaries (stepper.cpp:202-247) for the axes in axis_mask (bit a),
 * `layers` ghost layers (1..4). */
int ppmlr_gpu_block_fill_boundaries(ppmlr_gpu_block* b, int axis_mask, int layers);
/* sweep_axis (stepper.cpp:249-282). */
int ppmlr_gpu_block_sweep(ppmlr_gpu_block* b, int axis, double dt);
/* apply_sources (stepper.cpp:141-200). */
int ppmlr_gpu_block_sources(ppmlr_gpu_block* b, double dt);
/* restore_frozen_core (stepper.cpp:284-286). */
int ppmlr_gpu_block_restore_frozen(ppmlr_gpu_block* b);
/* Harness::advance for a whole-domain (1,1,1) block: global dt, the XYZ/ZYX
 * sweeps with boundary fills, sources, frozen core.  Runs as a CUDA graph.
 * *dt_out (may be NULL) receives the dt used. */
int ppmlr_gpu_block_advance(ppmlr_gpu_block* b, double cfl, int with_sources, long step,
                            double* dt_out);
/* `steps` consecutive advances starting at `first_step` without host
 * synchronisation; errors are checked once at the end (the first failure in
 * step order is reported).  *time_out (may be NULL) += sum of dts. */
int ppmlr_gpu_block_run(ppmlr_gpu_block* b, double cfl, int with_sources, long first_step,
                        long steps, double* time_out);

/* Halo exchange pieces (exchange.cpp:30-82).  face 0..5 = -x,+x,-y,+y,-z,+z.
 * pack: the `layers` outermost interior layers of `face` into dev_buf in the
 * reference HaloSlab order (t2 -> t1 -> layer -> 8 scalars).  unpack: writes
 * a slab packed by the neighbour's opposite face into this block's ghost
 * shell on `face`.  dev_buf is device memory on the block's device. */
int ppmlr_gpu_block_pack_face(ppmlr_gpu_block* b, int face, int layers, double* dev_buf);
int ppmlr_gpu_block_unpack_face(ppmlr_gpu_block* b, int face, int layers,
                                const double* dev_buf);
/* In-process exchange without staging: dst's ghost shell on `face` <- the
 * `layers` outermost interior layers of src's opposite face. */
int ppmlr_gpu_block_copy_face(ppmlr_gpu_block* dst, int face, ppmlr_gpu_block* src,
                              int layers);
/* Stream-ordered pieces of Harness::advance for an external (multi-process)
 * driver that owns the halo exchange and the dt reduction:
 *   begin:      reset the error window; dt slot <- this block's cfl*min
 *               (then min-reduce the dt slot across ranks)
 *   sweep_async: sweep_axis along `axis` as sweep number order_index (0..2)
 *               of the step, dt from the dt slot; ghosts must be current
 *   end_step:   apply_sources (+frozen core) or the frozen core alone, close
 *               the step (time += dt) and put the next local cfl*min in
 *               the dt slot (min-reduce it again before the next step)
 * Errors are reported by ppmlr_gpu_block_check(). */
int ppmlr_gpu_block_begin(ppmlr_gpu_block* b, double cfl, long first_step);
int ppmlr_gpu_block_sweep_async(ppmlr_gpu_block* b, int axis, int order_index);
int ppmlr_gpu_block_end_step(ppmlr_gpu_block* b, double cfl, int with_sources);
/* Split launches for overlapping a halo exchange with the producing kernel:
 * part 1 updates only the tiles that hold the 4 x-boundary cells of either
 * side (what an x neighbour reads), part 2 the rest; issue part 1, pack and
 * send the faces, then part 2 (which completes the sweep / the step).
 * part 0 = the whole launch (sweep_async / end_step). */
int ppmlr_gpu_block_sweep_part(ppmlr_gpu_block* b, int axis, int order_index, int part);
int ppmlr_gpu_block_end_step_part(ppmlr_gpu_block* b, double cfl, int with_sources, int part);
/* Simulated time accumulated on the device (host sync). */
int ppmlr_gpu_block_time(ppmlr_gpu_block* b, double* time_out);
/* Device scalars for external drivers (e.g. an NCCL min all-reduce of dt):
 * the block's dt slot (double) used by sweeps/sources issued with dt < 0. */
double* ppmlr_gpu_block_dt_slot(ppmlr_gpu_block* b);
/* Local CFL candidate cfl*min into the dt slot, asynchronously. */
int ppmlr_gpu_block_local_dt_async(ppmlr_gpu_block* b, double cfl);
/* cudaStream_t the block issues on (as void*), and setting it. */
void* ppmlr_gpu_block_stream(ppmlr_gpu_block* b);
int ppmlr_gpu_block_set_stream(ppmlr_gpu_block* b, void* stream);
int ppmlr_gpu_block_synchronize(ppmlr_gpu_block* b);
/* Device-resident state of the block (no copy; valid until the next call
 * that steps or uploads): the 8 field planes (rho, vx, vy, vz, Bx', By',
 * Bz', p) of the current buffer, each S0 x S1 x S2 ghost-inclusive with
 * element strides (1, strides[1], strides[2]); dims = S.  Returns the device
 * ghost width (4).  For on-device consumers (analysis, comparisons). */
int ppmlr_gpu_block_state_view(ppmlr_gpu_block* b, double** field_planes, long long* strides,
                               int* dims);
/* init_with of a built-in IC (kinds 0..3, see ppmlr_gpu_harness_init_ic)
 * evaluated on the device for this block (and its dipole, when it has one):
 * no host arrays, bit-identical to the host evaluation.  Clears the frozen
 * core. */
int ppmlr_gpu_block_init_ic(ppmlr_gpu_block* b, int kind, const double* params);
/* The dipole field B_d (3 planes, same layout as the state) or NULLs;
 * returns 1 when the block carries one.  Read-only: the y/z sweeps read
 * brick copies of B_d built at upload / init (change B_d via upload). */
int ppmlr_gpu_block_dipole_view(ppmlr_gpu_block* b, double** bd_planes);
/* Error word check (host sync): returns the status of the first failure
 * recorded since the last check, with the reference's message. */
int ppmlr_gpu_block_check(ppmlr_gpu_block* b);

/* Kernel-timing hooks for benchmarks.  While enabled, advance/run launch
 * kernels directly (no graph) and bracket every sweep kernel with CUDA
 * events on the block's stream (no host synchronisation).  A call returns
 * the summed sweep-kernel milliseconds, the number of timed sweep launches
 * and the number of kernels the block enqueued since the previous call,
 * then resets and sets the enable state. */
int ppmlr_gpu_block_timing(ppmlr_gpu_block* b, int enable, double* sweep_ms,
                           double* kernels_enqueued, long* sweep_launches);

/* ------------------------------------------------------------------------
 * Minimum slice: sweep_1d (ppm1d.cpp:317-364) over a batch of independent
 * strips with shared spacings.  states: nstrips x (n+2g) x 8 AoS (in/out,
 * interiors updated), bd: nstrips x (n+2g) x 3 or NULL, dx: n+2g.
 * ---------------------------------------------------------------------- */
int ppmlr_gpu_sweep_strips(double* states, const double* bd, const double* dx, int n,
                           int ghost, int nstrips, int dir, double dt, double gamma,
                           double mu0, double pressure_floor, int precision, int device);
/* strip_max_dt (ppm1d.cpp:307-315): min over the strips' interior cells of
 * dx / (|v_dir| + c_f,dir), bit-identical to the reference (IEEE ops). */
int ppmlr_gpu_strip_max_dt(const double* states, const double* bd, const double* dx, int n,
                           int ghost, int nstrips, int dir, double gamma, double mu0,
                           int device, double* dt_out);

/* ------------------------------------------------------------------------
 * Harness (harness.hpp:48-87): all blocks of a layout in one process (each
 * on `device`), exchanges as device-to-device copies, ledger kept with the
 * reference's accounting.
 * ---------------------------------------------------------------------- */
typedef struct ppmlr_gpu_harness ppmlr_gpu_harness;

struct ppmlr_gpu_options {
  double cfl;
  int ghost;
  int boundary;   /* PPMLR_BC_* */
  int transport;  /* 0 staged, 1 direct (ledger accounting only) */
  int with_sources, with_dipole;
  double wind_rho, wind_p, wind_v[3], wind_imf[3];
  double mu0, gamma, pressure_floor;
  int precision;
  int device;
}; /* HarnessOptions, harness.hpp:34-43 */

int ppmlr_gpu_harness_create(const ppmlr_axis_spec specs[3], int px, int py, int pz,
                             const ppmlr_gpu_options* opts, ppmlr_gpu_harness** out);
/* The same harness over several GPUs of one process: block r lives on
 * devices[r % ndevices] (peer access is enabled between them; creation fails
 * with PPMLR_RUNTIME when a pair has none).  Each block issues on its own
 * stream; halo copies pull the neighbours' faces over NVLink after their
 * state events and the global dt is a min over the blocks' device slots, so
 * a step has no host synchronisation (harness.hpp:79 / harness.cpp:18-28:
 * the reference keeps every rank in one process too). */
int ppmlr_gpu_harness_create_on(const ppmlr_axis_spec specs[3], int px, int py, int pz,
                                const ppmlr_gpu_options* opts, const int* devices,
                                int ndevices, ppmlr_gpu_harness** out);
void ppmlr_gpu_harness_destroy(ppmlr_gpu_harness* h);
/* init_magnetosphere (harness.cpp:30-33, stepper.cpp:83-112) */
int ppmlr_gpu_harness_init_magnetosphere(ppmlr_gpu_harness* h, double rho_core,
                                         double p_core, double falloff, double r_ref);
/* init_with (harness.cpp:35-43) for the built-in synthetic ICs:
 * 0 uniform(params = rho,vx,vy,vz,bx,by,bz,p), 1 Brio-Wu, 2 Orszag-Tang
 * (params[0] = gamma), 3 blast per unit block (p_in, p_out, radius),
 * 4 partition_ic (verify.cpp:195-203), 5 smooth_ic (acceptance.cpp:59-65),
 * 6 conservation gaussian (verify.cpp:165-169). */
int ppmlr_gpu_harness_init_ic(ppmlr_gpu_harness* h, int kind, const double* params);
/* init_with from caller-evaluated states: one ghost-inclusive AoS array per
 * block, concatenated in rank order. */
int ppmlr_gpu_harness_set_state(ppmlr_gpu_harness* h, const double* fields_all);
int ppmlr_gpu_harness_compute_dt(ppmlr_gpu_harness* h, double* dt_out);
int ppmlr_gpu_harness_advance(ppmlr_gpu_harness* h, double* dt_out);
int ppmlr_gpu_harness_run(ppmlr_gpu_harness* h, long steps);
/* gather_interior (harness.cpp:98-114): nx*ny*nz*8 AoS, x fastest. */
int ppmlr_gpu_harness_gather(ppmlr_gpu_harness* h, double* out);
long ppmlr_gpu_harness_step_count(ppmlr_gpu_harness* h);
double ppmlr_gpu_harness_time(ppmlr_gpu_harness* h);
int ppmlr_gpu_harness_block_count(ppmlr_gpu_harness* h);
ppmlr_gpu_block* ppmlr_gpu_harness_block(ppmlr_gpu_harness* h, int rank);
/* TransferLedger totals (exchange.hpp:48-61): bytes, messages, copy events. */
void ppmlr_gpu_harness_ledger(ppmlr_gpu_harness* h, uint64_t* bytes, long* messages,
                              long* copy_events);
/* TransferLedger entries (one per exchange_step, exchange.cpp:93-149):
 * returns the count and fills at most `max` of each array (any may be NULL).
 * transport: 0 staged, 1 direct. */
long ppmlr_gpu_harness_ledger_entries(ppmlr_gpu_harness* h, long* step, int* transport,
                                      long* messages, uint64_t* bytes, long* copy_events,
                                      long max);
/* write_snapshot(path, make_snapshot(h)) (src/snapshot.cpp:58-85,
 * tools/ppmlr_main.cpp:20-31): the PPLR v1 file of the current state.
 * _begin captures the state on the device and returns; a host thread drains
 * it to the file while the caller keeps stepping.  _wait joins and returns
 * the writer's status (InvalidSpec "snapshot: cannot open for writing: ..."
 * like the reference).  ppmlr_gpu_harness_snapshot = begin + wait. */
int ppmlr_gpu_harness_snapshot_begin(ppmlr_gpu_harness* h, const char* path);
int ppmlr_gpu_harness_snapshot_wait(ppmlr_gpu_harness* h);
int ppmlr_gpu_harness_snapshot(ppmlr_gpu_harness* h, const char* path);
/* Frozen-core record of block r (count if idx == NULL). */
int64_t ppmlr_gpu_harness_frozen(ppmlr_gpu_harness* h, int rank, int64_t* idx,
                                 double* states);
/* Ghost-inclusive geometry and dipole of block r (as make_block builds it). */
int ppmlr_gpu_harness_block_geometry(ppmlr_gpu_harness* h, int rank, int* n, int* lo,
                                     double* centers_cat, double* spacings_cat,
                                     double* bd /* or NULL */);

#ifdef __cplusplus
}
#endif
#endif
