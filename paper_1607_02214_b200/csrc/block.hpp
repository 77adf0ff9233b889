// Internal definition of a device-resident block (BlockState on one B200).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "../../include/ppmlr_gpu.h"
#include "ppmlr_common.hpp"

namespace ppmlr_b200 {


// Per-axis device geometry, ghost-inclusive with kG ghosts (span = n + 8).
struct DevAxis {
  double* dx = nullptr;     // spacings
  double* slope = nullptr;  // 3 per position: limited_slope coefficients
  double* qfc = nullptr;    // 5 per edge: interface-value coefficients
  double* hm = nullptr;     // centers[l] - centers[l-1]   (apply_sources)
  double* hp = nullptr;     // centers[l+1] - centers[l]
  double* rdx = nullptr;    // rcp_refined(dx)            (exact-division helper)
  double* den = nullptr;    // (hm*hp)*(hm+hp)            (central_diff denominator)
  double* rden = nullptr;   // rcp_refined(den)
  int span = 0;
};

struct SweepTiming {
  bool enabled = false;
  std::vector<cudaEvent_t> pool;  // pairs (start, end) per sweep launch
  size_t used = 0;                // events consumed in the pool
  double sweep_ms = 0.0, total_ms = 0.0;
  long launches = 0;              // sweep launches timed
};

struct StepGraph {
  cudaGraphExec_t exec = nullptr;
  int parity = -1;
  int with_sources = -1;
  int cur = -1;
  double cfl = -1.0;
};

}  // namespace ppmlr_b200

namespace ppmlr_b200 {
struct SweepMaps;
struct SrcMaps;
}

struct ppmlr_gpu_block {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  int n[3] = {0, 0, 0};
  int lo[3] = {0, 0, 0};
  int g_ref = 4;             // ghost width of the caller's arrays
  int S[3] = {0, 0, 0};      // n + 8
  int P0 = 0;                // padded x pitch (>= S[0], multiple of 8)
  long long sx = 1, sy = 0, sz = 0;
  long long ncell = 0;       // elements of the arena (both buffers + B_d)
  long long fs = 0;          // field stride: planar S[2]*sz, row-interleaved P0
  double* arena = nullptr;   // one allocation: buf[0], buf[1], bd
  double* buf[2] = {nullptr, nullptr};  // 8 fields each
  int cur = 0;               // buffer holding the current state
  double* bd = nullptr;      // 3 planes or nullptr
  double* bdz[2] = {nullptr, nullptr};  // B_d bricks for the y / z sweeps (SweepArgs::bdz)
  long long bdz_cs[2] = {0, 0};         // elements per brick component
  int bdz_ngx = 0;           // x groups of 4 interior cells
  bool bd_dirty = false;     // bd written since the bricks were built
  ppmlr_b200::DevAxis ax[3];
  std::vector<double> h_centers[3], h_spacings[3];  // kG-ghost windows
  int physical[3][2] = {{0, 0}, {0, 0}, {0, 0}};
  ppmlr_b200::Consts c{};
  int boundary = 0;
  double wind[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  bool with_dipole = false;
  int precision = PPMLR_STRICT;
  std::string deferred_error;  // e.g. periodic on a partial axis (apply_boundaries)
  int deferred_code = 0;
  // frozen inner core: bounding box + slot map
  long long n_frozen = 0;
  int fbox_lo[3] = {0, 0, 0}, fbox_n[3] = {0, 0, 0};
  int* fslot = nullptr;        // fbox volume, -1 = not frozen
  double* fstates = nullptr;   // 8 planes of n_frozen
  long long* fidx = nullptr;   // device linear indices (for the standalone restore)
  // device scalars
  unsigned long long* d_err = nullptr;   // first-failure key
  unsigned* d_redo = nullptr;            // [0] count, [1..] tiles/cells re-run exactly
  unsigned redo_cap = 0;
  unsigned long long* d_step = nullptr;  // step counter for keys (relative)
  unsigned long long* d_min = nullptr;   // CFL min as ordered bits
  double* d_dt = nullptr;                // dt in use
  double* d_dt_prev = nullptr;           // dt of the last completed step
  double* d_time = nullptr;              // accumulated time
  double* h_pinned = nullptr;            // 8 doubles pinned scratch
  long step_base = 0;                    // absolute step of d_step == 0
  double* d_scratch = nullptr;           // staging for upload/download
  cudaStream_t copy_stream = nullptr;    // host<->device chunk copies, overlapped with the
                                         // layout-conversion kernels on `stream`
  size_t scratch_bytes = 0;
  ppmlr_b200::StepGraph graphs[2][2];    // [parity][cur]
  ppmlr_b200::SweepTiming timing;
  cudaEvent_t ev[8] = {};
  long kernel_launches = 0;              // every kernel this block enqueued
  int sweep_L[3] = {0, 0, 0};            // segment length per axis
  int sweep_threads[3] = {0, 0, 0};
  // snapshot (gather_interior -> write_snapshot): a device copy of the
  // interior, field-major and x fastest like the PPLR payload, drained to
  // the host on its own stream while stepping continues
  double* d_snap = nullptr;
  cudaStream_t snap_stream = nullptr;
  cudaEvent_t snap_ready = nullptr;
  // TMA descriptors of the sweep inputs: [source buffer][axis] (block.cu)
  ppmlr_b200::SweepMaps* maps = nullptr;
  ppmlr_b200::SrcMaps* src_maps = nullptr;  // [source buffer]
  // The last run/advance left the next step's dt (cfl * fused CFL min of
  // the current state) in the device slot: the next run skips its
  // standalone CFL pass.  Any other state change clears it.
  bool dt_valid = false;
  double dt_cfl = 0.0;
};

namespace ppmlr_b200 {
void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
// Launchers implemented in sweep_*.cu
struct SweepArgs;
struct SweepMaps;
cudaError_t launch_sweep_strict(int axis, bool dipole, const SweepArgs& a, const SweepMaps& m,
                                int threads, size_t smem, cudaStream_t st);
struct SrcArgs;
struct SrcMaps;
cudaError_t launch_sources_strict(const SrcArgs& a, const SrcMaps& m, bool dipole,
                                  cudaStream_t st);
cudaError_t launch_sources_fast(const SrcArgs& a, const SrcMaps& m, bool dipole,
                                cudaStream_t st);
cudaError_t launch_sweep_fast(int axis, bool dipole, const SweepArgs& a, const SweepMaps& m,
                              int threads, size_t smem, cudaStream_t st);
}  // namespace ppmlr_b200

namespace ppmlr_b200 {
// Stream-ordered building blocks of a step (block.cu); used by the harness.
// part: 0 every tile, 1 the tiles holding the 4 x-boundary cells of either
// side, 2 the other tiles (grid_types.cuh split_*).  Parts 0 and 1 flip
// b->cur (after part 1 the current buffer holds the new boundary cells, so
// the faces can be packed); part 2 reads the other buffer and completes it.
int launch_sweep(ppmlr_gpu_block* b, int axis, int phase, int part = 0);
int launch_bc(ppmlr_gpu_block* b, int axis_mask, int layers);
int launch_sources(ppmlr_gpu_block* b, int fuse_cfl, int part = 0);  // same parts
int launch_frozen(ppmlr_gpu_block* b);
int launch_cfl(ppmlr_gpu_block* b, unsigned long long step_add);
int launch_step_end(ppmlr_gpu_block* b, double cfl, int close_step, int have_min);
int block_set_dt(ppmlr_gpu_block* b, double dt);  // dt < 0: keep the device slot

// Streamed state upload (block.cu).  `fill(kr0, nk, fields, bd)` writes the
// reference-layout (ghost g_ref) AoS k-planes [kr0, kr0 + nk): 8 doubles per
// cell into `fields`, 3 per cell into `bd` when `bd` is non-null.
using ChunkFill = std::function<void(int kr0, int nk, double* fields, double* bd)>;
int block_set_frozen(ppmlr_gpu_block* b, const int64_t* frozen_idx, const double* frozen_states,
                     int64_t n_frozen);
// With src_fields (and src_bd) given, chunks are copied straight from those
// caller buffers and `fill` is unused.
int block_upload_streamed(ppmlr_gpu_block* b, const ChunkFill& fill, bool with_bd,
                          const double* src_fields = nullptr, const double* src_bd = nullptr);
int block_finish_upload(ppmlr_gpu_block* b);
// Device-side setup (make_block default + dipole, init_with kinds 0..3),
// bit-identical to the host path; frozen set untouched.
bool device_init_supported(int kind);
int block_init_device(ppmlr_gpu_block* b, int kind, const double* params, bool with_bd);
// Multi-block harness plumbing (block.cu): the global-dt reduction over the
// blocks' device slots, and the error window / first-failure key of a block.
int launch_dt_min_all(double* const* d_slots, int n, cudaStream_t st);
int block_begin_window(ppmlr_gpu_block* b, long first_step);
int block_read_error(ppmlr_gpu_block* b, unsigned long long* key, unsigned long long* step);
int block_reset_error(ppmlr_gpu_block* b);
int block_last_dt_time(ppmlr_gpu_block* b, double* dt, double* time);  // host sync
int block_raise_error(ppmlr_gpu_block* b, unsigned long long key);
}  // namespace ppmlr_b200
