// Kernel-argument types shared by the block runtime (block.cu) and the
// precision-specific stencil translation units (sources_*.cu).
#pragma once
#include <cuda_runtime.h>

#include "ppmlr_common.hpp"

namespace ppmlr_b200 {

constexpr unsigned long long kInfBits = 0x7FF0000000000000ull;

struct Lay {
  int n0, n1, n2;
  int P0, S1;
  long long sy, sz, fs;  // y / z cell strides; fs: distance between two fields
  __host__ __device__ long long idx(int i, int j, int k) const {  // interior coords
    return (long long)(i + kG) + sy * (j + kG) + sz * (k + kG);
  }
};

struct Planes {
  double* f[8];
};

struct CtxPtrs {
  unsigned long long* err;
  unsigned long long* step;
  unsigned long long* min;
  double* dt;
  double* dt_prev;
  double* time;
};

__device__ __forceinline__ void cross3(double ax, double ay, double az, double bx, double by,
                                       double bz, double* o) {
  o[0] = ay * bz - az * by;
  o[1] = az * bx - ax * bz;
  o[2] = ax * by - ay * bx;
}

__device__ __forceinline__ void block_min_commit(double mn, unsigned long long* gmin) {
  // positive doubles order like their bit patterns
  unsigned long long bits = __double_as_longlong(mn);
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, bits, o);
    bits = other < bits ? other : bits;
  }
  __shared__ unsigned long long wmin[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) wmin[w] = bits;
  __syncthreads();
  if (w == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    bits = lane < nw ? wmin[lane] : kInfBits;
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, bits, o);
      bits = other < bits ? other : bits;
    }
    if (lane == 0 && bits != kInfBits) atomicMin(gmin, bits);
  }
}

// Split launches for the halo overlap: a launch over `count` x units (sweep
// segments / pencil groups / source x tiles) of part 1 covers the boundary
// units [0, cl) and [cr, count), part 2 the interior [cl, cr), part 0 all.
__host__ __device__ __forceinline__ int split_count(int part, int cl, int cr, int count) {
  return part == 1 ? cl + (count - cr) : (part == 2 ? cr - cl : count);
}
__host__ __device__ __forceinline__ int split_unit(int part, int cl, int cr, int u) {
  return part == 1 ? (u < cl ? u : cr + (u - cl)) : (part == 2 ? cl + u : u);
}

}  // namespace ppmlr_b200
