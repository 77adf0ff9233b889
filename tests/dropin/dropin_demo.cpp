// Drop-in check through the C++ API (TEST INFRASTRUCTURE: links the
// reference build under oracle/_ref as the comparison).  The reference's
// own RunConfig drives ppmlr::Harness on the CPU and GpuHarness on the GPU
// side by side; every dt and the final interior must be bit-identical.
//   usage: dropin_demo [steps] [px] [ndevices]
// ndevices > 1 maps the blocks round-robin onto that many device slots
// (ppmlr_gpu_harness_create_on); on a one-GPU box every slot is device 0,
// which runs the same multi-device code path.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cuda_runtime.h>

#include <vector>

#include "gpu_harness.hpp"
#include "ppmlr/decomp.hpp"

int main(int argc, char** argv) {
  using namespace ppmlr;
  const long steps = argc > 1 ? std::atol(argv[1]) : 4;
  RunConfig cfg;  // magnetosphere physics (dipole, sunward inflow, frozen core)
  cfg.grid_x = {-48.0, 28.8, -48.0, 28.8, 1.2, 64, 1.05};
  cfg.grid_y = {-21.6, 21.6, -21.6, 21.6, 1.2, 36, 1.05};
  cfg.grid_z = cfg.grid_y;
  cfg.partition.nx = argc > 2 ? std::atoi(argv[2]) : 2;
  try {
    const StretchedGrid grid = cfg.make_grid();
    Harness cpu(grid, layout(cfg.partition, grid), cfg.make_options());
    cpu.init_magnetosphere(cfg.profiles);
    const int ndev = argc > 3 ? std::atoi(argv[3]) : 1;
    int have = 1;
    cudaGetDeviceCount(&have);
    std::vector<int> devs;
    for (int d = 0; d < ndev; ++d) devs.push_back(d % (have > 0 ? have : 1));
    GpuHarness gpu(cfg, PPMLR_STRICT, devs);
    gpu.init_magnetosphere(cfg.profiles);
    for (long s = 0; s < steps; ++s) {
      const double a = cpu.advance(), b = gpu.advance();
      if (std::memcmp(&a, &b, sizeof a) != 0) {
        std::printf("dt differs at step %ld: %.17g vs %.17g\n", s, a, b);
        return 1;
      }
    }
    const auto x = cpu.gather_interior(), y = gpu.gather_interior();
    if (x.size() != y.size() || std::memcmp(x.data(), y.data(), x.size() * sizeof x[0]) != 0) {
      std::printf("state differs after %ld steps\n", steps);
      return 1;
    }
    std::printf("drop-in OK: %ld steps, partition (%d,1,1) on %d device slot(s), dt and %zu "
                "cells bit-identical\n",
                steps, cfg.partition.nx, ndev, x.size());
    return 0;
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
    return 2;
  }
}
