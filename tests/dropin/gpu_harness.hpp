// The maintainer-side binding of INTEGRATION.md, compiled: a drop-in for
// ppmlr::Harness (include/ppmlr/harness.hpp:48-87) on the GPU path through
// the C-ABI of include/ppmlr_gpu.h.  Header-only; link -lppmlr_b200.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "ppmlr/config.hpp"
#include "ppmlr/errors.hpp"
#include "ppmlr/harness.hpp"
#include "ppmlr_gpu.h"

namespace ppmlr {

inline void gpu_check(int rc) {
  if (rc == 0) return;
  const std::string m = ppmlr_gpu_last_error();
  switch (rc) {
    case PPMLR_INVALID_SPEC: throw InvalidSpec(m);
    case PPMLR_UNPHYSICAL: throw UnphysicalState(m);
    case PPMLR_STEP_REJECTED: throw StepRejected(m);
    case PPMLR_OUT_OF_RANGE: throw OutOfRange(m);
    default: throw Error(m);
  }
}

class GpuHarness {
 public:
  explicit GpuHarness(const RunConfig& cfg, int precision = PPMLR_STRICT, int device = 0)
      : GpuHarness(cfg, precision, std::vector<int>{device}) {}
  // One process driving several GPUs: block r on devices[r % size]
  // (ppmlr_gpu_harness_create_on; e.g. {0,1,...,7} for the 8 GPUs of a box).
  GpuHarness(const RunConfig& cfg, int precision, const std::vector<int>& devices) {
    ppmlr_axis_spec s[3];
    const AxisSpec* a[3] = {&cfg.grid_x, &cfg.grid_y, &cfg.grid_z};
    for (int i = 0; i < 3; ++i)
      s[i] = {a[i]->min,      a[i]->max,          a[i]->uniform_lo, a[i]->uniform_hi,
              a[i]->d_uniform, a[i]->target_cells, a[i]->nominal_ratio};
    ppmlr_gpu_options o{};
    o.cfl = cfg.cfl;
    o.ghost = cfg.ghost;
    o.boundary = static_cast<int>(cfg.boundary);  // Outflow, Periodic, Magnetosphere
    o.transport = cfg.transport == TransportKind::Direct ? 1 : 0;
    o.with_sources = cfg.with_sources;
    o.with_dipole = cfg.with_dipole;
    o.wind_rho = cfg.wind.rho_sw;
    o.wind_p = cfg.wind.p_sw;
    for (int i = 0; i < 3; ++i) {
      o.wind_v[i] = cfg.wind.v_sw[i];
      o.wind_imf[i] = cfg.wind.imf[i];
    }
    o.mu0 = cfg.constants.mu0;
    o.gamma = cfg.constants.gamma;
    o.pressure_floor = cfg.constants.pressure_floor;
    o.precision = precision;  // PPMLR_STRICT: bit-identical to the CPU build
    o.device = devices.empty() ? 0 : devices[0];
    gpu_check(ppmlr_gpu_harness_create_on(s, cfg.partition.nx, cfg.partition.ny,
                                          cfg.partition.nz, &o, devices.data(),
                                          static_cast<int>(devices.size()), &h_));
    cells_ = static_cast<std::size_t>(cfg.grid_x.target_cells) * cfg.grid_y.target_cells *
             cfg.grid_z.target_cells;
  }
  ~GpuHarness() { ppmlr_gpu_harness_destroy(h_); }
  GpuHarness(GpuHarness&& o) noexcept : h_(o.h_), cells_(o.cells_) { o.h_ = nullptr; }
  GpuHarness(const GpuHarness&) = delete;
  GpuHarness& operator=(const GpuHarness&) = delete;

  void init_magnetosphere(const InitialProfiles& p) {
    gpu_check(ppmlr_gpu_harness_init_magnetosphere(h_, p.rho_core, p.p_core, p.falloff, p.r_ref));
  }
  double compute_global_dt() const {
    double dt;
    gpu_check(ppmlr_gpu_harness_compute_dt(h_, &dt));
    return dt;
  }
  double advance() {
    double dt;
    gpu_check(ppmlr_gpu_harness_advance(h_, &dt));
    return dt;
  }
  void run(long steps) { gpu_check(ppmlr_gpu_harness_run(h_, steps)); }
  long step_count() const { return ppmlr_gpu_harness_step_count(h_); }
  double time() const { return ppmlr_gpu_harness_time(h_); }
  std::vector<PrimitiveState> gather_interior() const {
    std::vector<PrimitiveState> out(cells_);  // 8 contiguous doubles each
    gpu_check(ppmlr_gpu_harness_gather(h_, reinterpret_cast<double*>(out.data())));
    return out;
  }
  void write_snapshot(const std::string& path) {  // ppmlr run cadence output
    gpu_check(ppmlr_gpu_harness_snapshot(h_, path.c_str()));
  }

 private:
  ppmlr_gpu_harness* h_ = nullptr;
  std::size_t cells_ = 0;
};

}  // namespace ppmlr
