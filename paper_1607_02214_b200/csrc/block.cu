// Device-resident block: state upload/download, boundary fills, CFL
// reduction, dipole source terms, frozen core, halo pack/unpack and the
// per-step CUDA graph.  Compiled with --fmad=false so every arithmetic
// kernel here is bit-identical to the reference (proj/src/stepper.cpp).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "block.hpp"
#include "sources.cuh"
#include "sweep.cuh"

using namespace ppmlr_b200;
using namespace ppmlr_b200::strict;

namespace ppmlr_b200 {

thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int cuda_fail(cudaError_t e, const char* where) {
  set_error(std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e));
  return PPMLR_RUNTIME;
}

}  // namespace ppmlr_b200

#define CK(call)                                              \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);       \
  } while (0)

namespace {

Lay lay_of(const ppmlr_gpu_block* b) {
  Lay l;
  l.n0 = b->n[0];
  l.n1 = b->n[1];
  l.n2 = b->n[2];
  l.P0 = b->P0;
  l.S1 = b->S[1];
  l.sy = b->sy;
  l.sz = b->sz;
  l.fs = b->fs;
  return l;
}

Planes planes(double* base, long long fs) {
  Planes p;
  for (int f = 0; f < 8; ++f) p.f[f] = base + f * fs;
  return p;
}

// ---------------------------------------------------------------- kernels



// ------------------------------------------------------------------ layout

// Reference AoS (ghost gr) k-plane chunk -> device SoA (ghost 4).
__global__ void aos_to_soa_kernel(const double* __restrict__ aos, int nper, Planes dst, Lay L,
                                  int gr, int S0r, int S1r, int kr0, int nk, const double* bdsrc,
                                  double* bd0, double* bd1, double* bd2) {
  const long long total = (long long)S0r * S1r * nk;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int ir = (int)(t % S0r);
    const int jr = (int)((t / S0r) % S1r);
    const int kr = kr0 + (int)(t / ((long long)S0r * S1r));
    const int i = ir - gr, j = jr - gr, k = kr - gr;
    if (i < -kG || i >= L.n0 + kG || j < -kG || j >= L.n1 + kG || k < -kG || k >= L.n2 + kG)
      continue;
    const long long d = L.idx(i, j, k);
    if (aos) {
      const double* s = aos + t * nper;
      for (int f = 0; f < 8; ++f) dst.f[f][d] = s[f];
    }
    if (bdsrc) {
      const double* s = bdsrc + t * 3;
      bd0[d] = s[0];
      bd1[d] = s[1];
      bd2[d] = s[2];
    }
  }
}

// Device SoA -> reference AoS (ghost gr) k-plane chunk.
__global__ void soa_to_aos_kernel(double* __restrict__ aos, Planes src, Lay L, int gr, int S0r,
                                  int S1r, int kr0, int nk) {
  const long long total = (long long)S0r * S1r * nk;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int ir = (int)(t % S0r);
    const int jr = (int)((t / S0r) % S1r);
    const int kr = kr0 + (int)(t / ((long long)S0r * S1r));
    const int i = ir - gr, j = jr - gr, k = kr - gr;
    double* o = aos + t * 8;
    if (i < -kG || i >= L.n0 + kG || j < -kG || j >= L.n1 + kG || k < -kG || k >= L.n2 + kG) {
      for (int f = 0; f < 8; ++f) o[f] = 0.0;
      continue;
    }
    const long long d = L.idx(i, j, k);
    for (int f = 0; f < 8; ++f) o[f] = src.f[f][d];
  }
}

// Interior only, x fastest.
// Interior of every field plane, field-major, x fastest (the PPLR payload
// order, snapshot.cpp:78-83): out[f * cells + i + n0 * (j + n1 * k)].
__global__ void interior_planes_kernel(double* __restrict__ out, Planes src, Lay L) {
  const long long total = (long long)L.n0 * L.n1 * L.n2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % L.n0);
    const int j = (int)((t / L.n0) % L.n1);
    const int k = (int)(t / ((long long)L.n0 * L.n1));
    const long long d = L.idx(i, j, k);
#pragma unroll
    for (int f = 0; f < 8; ++f) out[f * total + t] = src.f[f][d];
  }
}

// Interior k-planes [k0, k0 + nk) as AoS, x fastest (gather_interior order).
__global__ void soa_to_interior_kernel(double* __restrict__ out, Planes src, Lay L, int k0,
                                       int nk) {
  const long long total = (long long)L.n0 * L.n1 * nk;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % L.n0);
    const int j = (int)((t / L.n0) % L.n1);
    const int k = k0 + (int)(t / ((long long)L.n0 * L.n1));
    const long long d = L.idx(i, j, k);
    for (int f = 0; f < 8; ++f) out[t * 8 + f] = src.f[f][d];
  }
}

// apply_boundaries (stepper.cpp:202-247) for one axis, `layers` ghost layers,
// over the interior transverse span.  mode: 0 outflow, 1 periodic,
// 2 magnetosphere (the sunward +x shell is constant and pre-filled).
// One launch fills the faces of every axis in `axes` (packed 2 bits per
// entry, blockIdx.y selects the entry): the slabs of different axes are
// disjoint (interior transverse ranges only).
struct BcAxes {
  int axis[3], lo[3], hi[3];
};

__global__ void bc_kernel(Planes s, Lay L, BcAxes ax, int layers, int mode) {
  const int axis = ax.axis[blockIdx.y], phys_lo = ax.lo[blockIdx.y], phys_hi = ax.hi[blockIdx.y];
  const int na = axis == 0 ? L.n0 : (axis == 1 ? L.n1 : L.n2);
  const int nb = axis == 0 ? L.n1 : (axis == 1 ? L.n2 : L.n0);
  const int nc = axis == 0 ? L.n2 : (axis == 1 ? L.n0 : L.n1);
  // 32-bit index arithmetic (a face slab has < 2^31 cells: launch_bc)
  const int per_side = layers * nb * nc;
  const int total = 2 * per_side;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int side = t >= per_side;
    const int r = t - side * per_side;
    // layer fastest for axis 0 (contiguous), transverse fastest otherwise
    int layer, t1, t2;
    if (axis == 0) {
      const int rl = r / layers;
      layer = 1 + (r - rl * layers);
      t2 = rl / nb;
      t1 = rl - t2 * nb;
    } else if (axis == 1) {  // iterate x fastest: x = t2 (d axis)
      const int rn = r / nc;
      t2 = r - rn * nc;
      layer = 1 + rn / nb;
      t1 = rn - (layer - 1) * nb;
    } else {  // x = t1 (b axis)
      const int rn = r / nb;
      t1 = r - rn * nb;
      layer = 1 + rn / nc;
      t2 = rn - (layer - 1) * nc;
    }
    if (side == 0 && !phys_lo) continue;
    if (side == 1 && !phys_hi) continue;
    if (mode == 2 && axis == 0 && side == 1) continue;  // sunward inflow: pre-filled
    int cell[3], src[3];
    cell[(axis + 1) % 3] = src[(axis + 1) % 3] = t1;
    cell[(axis + 2) % 3] = src[(axis + 2) % 3] = t2;
    cell[axis] = side == 0 ? -layer : na - 1 + layer;
    if (mode == 1)
      src[axis] = side == 0 ? na - layer : layer - 1;
    else
      src[axis] = side == 0 ? 0 : na - 1;
    const long long d = L.idx(cell[0], cell[1], cell[2]);
    const long long q = L.idx(src[0], src[1], src[2]);
#pragma unroll
    for (int f = 0; f < 8; ++f) s.f[f][d] = s.f[f][q];
  }
}

// Sunward (+x) ghost shell in Magnetosphere mode: rho, v, p of the wind and
// B' = imf - bd(ghost)  (stepper.cpp:227-236).  Constant for the whole run.
__global__ void wind_fill_kernel(Planes s, Lay L, const double* bd0, const double* bd1,
                                 const double* bd2, double rho, double p, double v0, double v1,
                                 double v2, double i0, double i1, double i2) {
  const long long total = (long long)kG * L.n1 * L.n2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int layer = 1 + (int)(t % kG);
    const int j = (int)((t / kG) % L.n1);
    const int k = (int)(t / ((long long)kG * L.n1));
    const long long d = L.idx(L.n0 - 1 + layer, j, k);
    s.f[0][d] = rho;
    s.f[1][d] = v0;
    s.f[2][d] = v1;
    s.f[3][d] = v2;
    s.f[4][d] = i0 - (bd0 ? bd0[d] : 0.0);
    s.f[5][d] = i1 - (bd1 ? bd1[d] : 0.0);
    s.f[6][d] = i2 - (bd2 ? bd2[d] : 0.0);
    s.f[7][d] = p;
  }
}

// B_d planes -> y / z bricks (SweepArgs::bdz): one thread per brick element,
// the padding pencils of a partial last x group are zero.
// axis 1: o = z, strip position y; axis 2: o = y, strip position z.
__global__ void bd_bricks_kernel(double* __restrict__ bdz, const double* __restrict__ bd,
                                 long long fs, Lay L, int axis, int ngx, int s2, long long cs) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < 3 * cs;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / cs);
    const long long r = e - c * cs;
    const int p = (int)(r & 3);
    const long long rq = r >> 2;
    const int q = (int)(rq % s2);
    const long long ox = rq / s2;
    const int xg = (int)(ox % ngx), o = (int)(ox / ngx);
    const int x = xg * 4 + p;
    const long long yz = axis == 2 ? L.sy * (o + kG) + L.sz * q : L.sy * q + L.sz * (o + kG);
    bdz[e] = x < L.n0 ? bd[c * fs + (x + kG) + yz] : 0.0;
  }
}

// Standalone compute_dt over the interior; min into ctx.min.
template <bool DIPOLE>
__global__ void cfl_kernel(Planes s, Lay L, const double* bd0, const double* bd1,
                           const double* bd2, const double* dx0, const double* dx1,
                           const double* dx2, Consts cc, CtxPtrs ctx, unsigned long long step_add) {
  const KC c = make_kc(cc);
  const long long total = (long long)L.n0 * L.n1 * L.n2;
  double mn = __longlong_as_double(kInfBits);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % L.n0);
    const int j = (int)((t / L.n0) % L.n1);
    const int k = (int)(t / ((long long)L.n0 * L.n1));
    const long long d = L.idx(i, j, k);
    double q[8];
#pragma unroll
    for (int f = 0; f < 8; ++f) q[f] = s.f[f][d];
    int bad = 0;
    if (!cfl_cell(q, DIPOLE ? bd0[d] : 0.0, DIPOLE ? bd1[d] : 0.0, DIPOLE ? bd2[d] : 0.0,
                  dx0[i + kG], dx1[j + kG], dx2[k + kG], c, mn, bad))
      atomicMin(ctx.err, err_key(*ctx.step + step_add, kPhaseCfl, 0,
                                 ((unsigned long long)t * 3 + bad) << 2));
  }
  block_min_commit(mn, ctx.min);
}

// dt = cfl * min; optionally close the current step first.
__global__ void step_end_kernel(CtxPtrs ctx, double cfl, int close_step, int have_min) {
  if (close_step) {
    *ctx.time += *ctx.dt;
    *ctx.dt_prev = *ctx.dt;
    *ctx.step += 1;
  }
  if (have_min) {
    *ctx.dt = cfl * __longlong_as_double(*ctx.min);
    *ctx.min = kInfBits;
  }
}

// In-place refined reciprocals of a geometry table.
__global__ void rcp_table_kernel(double* v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = rcp_refined(v[i]);
}

__global__ void frozen_restore_kernel(Planes s, const long long* idx, const double* st,
                                      long long nf) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nf;
       t += (long long)gridDim.x * blockDim.x) {
    const long long d = idx[t];
#pragma unroll
    for (int f = 0; f < 8; ++f) s.f[f][d] = st[f * nf + t];
  }
}

// Face slab addressing (exchange.cpp:17-27): layer q of the face in global
// order; pack order t2 -> t1 -> layer -> 8 scalars.
__device__ __forceinline__ void face_cell(int axis, int t1, int t2, int along, int* cell) {
  cell[(axis + 1) % 3] = t1;
  cell[(axis + 2) % 3] = t2;
  cell[axis] = along;
}

__global__ void pack_kernel(Planes s, Lay L, int face, int layers, double* out) {
  const int axis = face / 2;
  const int na = axis == 0 ? L.n0 : (axis == 1 ? L.n1 : L.n2);
  const int nb = axis == 0 ? L.n1 : (axis == 1 ? L.n2 : L.n0);
  const int nc = axis == 0 ? L.n2 : (axis == 1 ? L.n0 : L.n1);
  // 32-bit index arithmetic: a face slab of >= 2^31 cells would need a
  // block beyond any GPU's memory
  const int total = nb * nc * layers;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int tl = t / layers;
    const int q = t - tl * layers;
    const int t2 = tl / nb;
    const int t1 = tl - t2 * nb;
    int cell[3];
    face_cell(axis, t1, t2, face % 2 == 0 ? q : na - layers + q, cell);
    const long long d = L.idx(cell[0], cell[1], cell[2]);
#pragma unroll
    for (int f = 0; f < 8; ++f) out[(long long)t * 8 + f] = s.f[f][d];
  }
}

// `face` is the receiver's face; the slab came from the sender's opposite face.
__global__ void unpack_kernel(Planes s, Lay L, int face, int layers, const double* in) {
  const int axis = face / 2;
  const int na = axis == 0 ? L.n0 : (axis == 1 ? L.n1 : L.n2);
  const int nb = axis == 0 ? L.n1 : (axis == 1 ? L.n2 : L.n0);
  const int nc = axis == 0 ? L.n2 : (axis == 1 ? L.n0 : L.n1);
  const int src_face = face ^ 1;
  // 32-bit index arithmetic: a face slab of >= 2^31 cells would need a
  // block beyond any GPU's memory
  const int total = nb * nc * layers;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int tl = t / layers;
    const int q = t - tl * layers;
    const int t2 = tl / nb;
    const int t1 = tl - t2 * nb;
    int cell[3];
    face_cell(axis, t1, t2, src_face % 2 == 0 ? na + q : -layers + q, cell);
    const long long d = L.idx(cell[0], cell[1], cell[2]);
#pragma unroll
    for (int f = 0; f < 8; ++f) s.f[f][d] = in[(long long)t * 8 + f];
  }
}

__global__ void copy_face_kernel(Planes dst, Lay Ld, Planes src, Lay Ls, int face, int layers) {
  const int axis = face / 2;
  const int nad = axis == 0 ? Ld.n0 : (axis == 1 ? Ld.n1 : Ld.n2);
  const int nas = axis == 0 ? Ls.n0 : (axis == 1 ? Ls.n1 : Ls.n2);
  const int nb = axis == 0 ? Ld.n1 : (axis == 1 ? Ld.n2 : Ld.n0);
  const int nc = axis == 0 ? Ld.n2 : (axis == 1 ? Ld.n0 : Ld.n1);
  const int src_face = face ^ 1;
  // 32-bit index arithmetic: a face slab of >= 2^31 cells would need a
  // block beyond any GPU's memory
  const int total = nb * nc * layers;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int tl = t / layers;
    const int q = t - tl * layers;
    const int t2 = tl / nb;
    const int t1 = tl - t2 * nb;
    int cs[3], cd[3];
    face_cell(axis, t1, t2, src_face % 2 == 0 ? q : nas - layers + q, cs);
    face_cell(axis, t1, t2, src_face % 2 == 0 ? nad + q : -layers + q, cd);
    const long long ds = Ls.idx(cs[0], cs[1], cs[2]);
    const long long dd = Ld.idx(cd[0], cd[1], cd[2]);
#pragma unroll
    for (int f = 0; f < 8; ++f) dst.f[f][dd] = src.f[f][ds];
  }
}

int grid_for(long long work, int threads = 256) {
  long long g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}

// ----------------------------------------------------------- host helpers

CtxPtrs ctx_of(ppmlr_gpu_block* b) {
  return CtxPtrs{b->d_err, b->d_step, b->d_min, b->d_dt, b->d_dt_prev, b->d_time};
}

double* cur_buf(ppmlr_gpu_block* b) { return b->buf[b->cur]; }

// State layout in HBM.  Both ping-pong buffers and B_d live in one arena,
// each field a [z][y][x] array with an x pitch P0 (default), or with
// PPMLR_LAYOUT=rows row-interleaved: for every (y, z) row the 8 fields of
// buffer 0, the 8 of buffer 1 and the 3 B_d components follow each other
// ([z][y][field][x], field stride P0, y stride NF*P0), so that a z-sweep
// tile touches 72 2 MB pages instead of 72 per field.  Measured (DESIGN.md
// §4): the C5 z sweep -2.4%, the blast 512^3 z sweep +18%; planar stays.
void set_state_layout(ppmlr_gpu_block* b) {
  b->P0 = ((b->S[0] + 7) / 8) * 8;
  const char* env = std::getenv("PPMLR_LAYOUT");
  const bool rows = env && std::strcmp(env, "rows") == 0;
  const long long nf = 16 + (b->with_dipole ? 3 : 0);
  if (!rows) {
    b->sy = b->P0;
    b->sz = (long long)b->P0 * b->S[1];
    b->fs = b->sz * b->S[2];
    b->ncell = nf * b->fs;
  } else {
    b->fs = b->P0;
    b->sy = nf * b->P0;
    b->sz = b->sy * b->S[1];
    b->ncell = b->sz * b->S[2];
  }
}

// buf[cur ^ 1] := buf[cur] (all 8 fields, ghosts included)
cudaError_t copy_state(ppmlr_gpu_block* b, double* dst, const double* src) {
  if (b->fs == b->P0)
    return cudaMemcpy2DAsync(dst, sizeof(double) * b->sy, src, sizeof(double) * b->sy,
                             sizeof(double) * 8 * b->P0, (size_t)b->S[1] * b->S[2],
                             cudaMemcpyDeviceToDevice, b->stream);
  return cudaMemcpyAsync(dst, src, sizeof(double) * 8 * b->fs, cudaMemcpyDeviceToDevice,
                         b->stream);
}

// Reference message for a decoded error key (sweep / sources / CFL).
int decode_error(ppmlr_gpu_block* b, unsigned long long key, std::string& msg) {
  const int phase = err_phase(key);
  const unsigned long long pos = err_pos(key);
  const int kind = (int)(pos & 3);
  char buf[512];
  if (phase == kPhaseCfl) {
    const unsigned long long cell = (pos >> 2) / 3;
    const int i = (int)(cell % b->n[0]);
    const int j = (int)((cell / b->n[0]) % b->n[1]);
    const int k = (int)(cell / ((unsigned long long)b->n[0] * b->n[1]));
    std::snprintf(buf, sizeof buf, "non-finite signal speed at cell (%d,%d,%d)", i, j, k);
    msg = buf;
    return PPMLR_UNPHYSICAL;
  }
  if (phase == kPhaseSources) {
    const unsigned long long cell = pos >> 2;
    const int i = (int)(cell % b->n[0]);
    const int j = (int)((cell / b->n[0]) % b->n[1]);
    const int k = (int)(cell / ((unsigned long long)b->n[0] * b->n[1]));
    std::snprintf(buf, sizeof buf, "%s after sources at cell (%d,%d,%d)",
                  kind == kErrDensity ? "non-positive density"
                                      : "non-positive pressure recovered from conserved state",
                  i, j, k);
    msg = buf;
    return PPMLR_UNPHYSICAL;
  }
  const int axis = err_axis(key);
  const unsigned long long pencil = pos >> 20;
  const int sub = (int)((pos >> 19) & 1);
  const int zone = (int)((pos >> 2) & 0x1FFFF);
  const int nb = b->n[(axis + 1) % 3];
  const int t1 = (int)(pencil % nb), t2 = (int)(pencil / nb);
  if (sub == 0) {
    if (kind == kErrStepRejected)
      std::snprintf(buf, sizeof buf, "Lagrangian interfaces crossed at zone %d", zone);
    else
      std::snprintf(buf, sizeof buf,
                    "negative density or pressure after Lagrangian step at zone %d", zone);
  } else {
    std::snprintf(buf, sizeof buf, "%s at strip cell %d",
                  kind == kErrDensity ? "non-positive density"
                                      : "non-positive pressure recovered from conserved state",
                  zone);
  }
  msg = buf;
  std::snprintf(buf, sizeof buf, " in sweep axis %d at line (%d,%d)", axis, t1, t2);
  msg += buf;
  return PPMLR_UNPHYSICAL;  // stepper.cpp:272-276 rethrows as UnphysicalState
}

void build_axis_tables(const std::vector<double>& dx, const std::vector<double>& ce,
                       std::vector<double>& slope, std::vector<double>& qfc,
                       std::vector<double>& hm, std::vector<double>& hp) {
  const int nn = (int)dx.size();
  slope.assign(3 * nn, 0.0);
  qfc.assign(5 * (nn + 1), 0.0);
  hm.assign(nn, 0.0);
  hp.assign(nn, 0.0);
  for (int k = 1; k + 1 < nn; ++k) {
    slope[3 * k] = dx[k] / ((dx[k - 1] + dx[k]) + dx[k + 1]);
    slope[3 * k + 1] = (2.0 * dx[k - 1] + dx[k]) / (dx[k + 1] + dx[k]);
    slope[3 * k + 2] = (dx[k] + 2.0 * dx[k + 1]) / (dx[k - 1] + dx[k]);
  }
  for (int m = 2; m + 1 < nn; ++m) {
    const int i = m - 1;
    double* e = &qfc[5 * m];
    e[0] = dx[i] / (dx[i] + dx[i + 1]);
    e[1] = 1.0 / (((dx[i - 1] + dx[i]) + dx[i + 1]) + dx[i + 2]);
    e[2] = (((2.0 * dx[i + 1]) * dx[i]) / (dx[i] + dx[i + 1])) *
           ((dx[i - 1] + dx[i]) / (2.0 * dx[i] + dx[i + 1]) -
            (dx[i + 2] + dx[i + 1]) / (2.0 * dx[i + 1] + dx[i]));
    e[3] = (dx[i] * (dx[i - 1] + dx[i])) / (2.0 * dx[i] + dx[i + 1]);
    e[4] = (dx[i + 1] * (dx[i + 1] + dx[i + 2])) / (dx[i] + 2.0 * dx[i + 1]);
  }
  for (int l = 1; l < nn; ++l) hm[l] = ce[l] - ce[l - 1];
  for (int l = 0; l + 1 < nn; ++l) hp[l] = ce[l + 1] - ce[l];
}

template <typename T>
int upload_vec(T** dst, const std::vector<T>& v) {
  CK(cudaMalloc(dst, sizeof(T) * std::max<size_t>(v.size(), 1)));
  CK(cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  return 0;
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

void choose_sweep_tiles(ppmlr_gpu_block* b) {
  // Segments of kSweepTL - 8 = 64 cells (compile-time tile) when the axis is a
  // multiple of 64 or long enough that a partial last segment costs little;
  // otherwise balanced segments of at most Lmax cells (runtime tile).
  // one cell per thread: a tile is at most kSweepNP * kSweepTL cells
  const int Lmax = std::min(env_int("PPMLR_SWEEP_LMAX", kSweepTL - 8), kSweepTL - 8);
  const int ipt = 1;
  const int Lc = kSweepTL - 8;
  for (int a = 0; a < 3; ++a) {
    const int n = b->n[a];
    int L;
    if (env_int("PPMLR_SWEEP_RUNTIME_TL", 0) == 0 &&
        (n % Lc == 0 || n >= 4 * Lc || env_int("PPMLR_SWEEP_FORCE_CT", 0))) {
      L = Lc;
    } else {
      const int nseg = (n + Lmax - 1) / Lmax;
      L = (n + nseg - 1) / nseg;
      L += L & 1;  // even: the x tile box row (TL doubles) must be a multiple of 16 B
      // fast build: the second compile-time tile (persistent kernel) when it
      // costs no more strip positions than the runtime tile, whose threads
      // round up to whole warps (C3 160/150: fast sweep 0.490 -> 0.478 ms;
      // strict 0.684 -> 0.705, so strict keeps the runtime tile)
      const int L2 = kSweepTL2 - 8;
      const int runtime_pos = nseg * ((kSweepNP * (L + 8) + 31) / 32 * 32) / kSweepNP;
      if (b->precision == PPMLR_FAST && env_int("PPMLR_SWEEP_RUNTIME_TL", 0) == 0 &&
          env_int("PPMLR_SWEEP_TL2_ON", 1) && (n + L2 - 1) / L2 * kSweepTL2 <= runtime_pos)
        L = L2;
    }
    b->sweep_L[a] = L;
    const int T = kSweepNP * (L + 8);
    int nt = (T + ipt - 1) / ipt;
    nt = ((nt + 31) / 32) * 32;
    b->sweep_threads[a] = std::min(kSweepNP * kSweepTL, std::max(32, nt));
  }
}

}  // namespace

// ------------------------------------------------------------------ sweeps

namespace ppmlr_b200 {

// The x-boundary split of a launch over `count` x units of `unit` cells.
static void split_range(int n0, int unit, int count, int& cl, int& cr) {
  cl = std::min(count, (kG + unit - 1) / unit);
  cr = std::max(cl, std::min(count, n0 >= kG ? (n0 - kG) / unit : 0));
}

int launch_sweep(ppmlr_gpu_block* b, int axis, int phase, int part) {
  SweepArgs A{};
  // part 1 flips b->cur at once (the neighbour faces are packed from the
  // new state before part 2 runs); part 2 then reads the other buffer
  const int src = part == 2 ? b->cur ^ 1 : b->cur;
  double* in = b->buf[src];
  double* out = b->buf[src ^ 1];
  for (int f = 0; f < 8; ++f) {
    A.src[f] = in + f * b->fs;
    A.dst[f] = out + f * b->fs;
  }
  for (int k = 0; k < 3; ++k) A.bd[k] = b->bd ? b->bd + k * b->fs : nullptr;
  A.bdz = axis > 0 ? b->bdz[axis - 1] : nullptr;
  A.bdz_cs = axis > 0 ? b->bdz_cs[axis - 1] : 0;
  A.bdz_ngx = b->bdz_ngx;
  A.bdz_s2 = b->S[axis];
  A.dx = b->ax[axis].dx;
  A.rdx = b->ax[axis].rdx;
  A.slope = b->ax[axis].slope;
  A.qfc = b->ax[axis].qfc;
  const long long strides[3] = {1, b->sy, b->sz};
  const int G = axis == 0 ? 1 : 0;
  const int O = axis == 2 ? 1 : 2;
  A.stride_a = strides[axis];
  A.stride_g = strides[G];
  A.stride_o = strides[O];
  A.n = b->n[axis];
  A.ng = b->n[G];
  A.no = b->n[O];
  A.nb = b->n[(axis + 1) % 3];
  A.L = b->sweep_L[axis];
  A.nseg = (A.n + A.L - 1) / A.L;
  A.ngroups = (A.ng + kSweepNP - 1) / kSweepNP;
  if (A.ngroups > 65535 || A.no > 65535) {  // grid (nseg, ngroups, no)
    set_error("sweep: too many pencils across the sweep axis for one launch grid");
    return PPMLR_INVALID_SPEC;
  }
  A.dt = b->d_dt;
  A.err = b->d_err;
  A.step = b->d_step;
  A.phase = phase;
  A.c = b->c;
  A.redo_count = b->d_redo;
  A.redo_list = b->d_redo + 1;
  A.tile_ctr = b->d_redo + b->redo_cap + 1;
  A.part = part;
  if (axis == 0)
    split_range(b->n[0], A.L, A.nseg, A.cl, A.cr);
  else
    split_range(b->n[0], kSweepNP, A.ngroups, A.cl, A.cr);
  const int T = slot_stride(kSweepNP * (A.L + 8));
  // shared slots per cell: 25 (+3 dipole), 33 with the extra-slot schedule
  // (sweep.cuh XS; with the dipole only in the strict build)
  const bool xs = PPMLR_SWEEP_XSLOTS &&
                  (!b->with_dipole ||
                   (b->precision == PPMLR_FAST ? PPMLR_SWEEP_XSD_FAST : PPMLR_SWEEP_XSD_STRICT));
  const int slots = xs ? 33 : (b->with_dipole ? 28 : 25);
  const size_t smem = sizeof(double) * (size_t)T * slots;
  // The sweep writes only the interior of the output buffer; its ghost
  // shells stay stale until the next fill (every reader fills first).
  cudaError_t e = b->precision == PPMLR_FAST
                      ? launch_sweep_fast(axis, b->with_dipole, A, b->maps[3 * src + axis],
                                          b->sweep_threads[axis], smem, b->stream)
                      : launch_sweep_strict(axis, b->with_dipole, A, b->maps[3 * src + axis],
                                            b->sweep_threads[axis], smem, b->stream);
  if (e != cudaSuccess) return cuda_fail(e, "sweep kernel launch");
  b->kernel_launches += 2;  // fast pass + exact re-run of flagged tiles
  if (part != 2) b->cur ^= 1;
  return 0;
}

int launch_bc(ppmlr_gpu_block* b, int axis_mask, int layers) {
  const Lay L = lay_of(b);
  Planes s = planes(cur_buf(b), b->fs);
  BcAxes ax{};
  int na = 0;
  long long work = 0;
  for (int a = 0; a < 3; ++a) {
    if (!(axis_mask & (1 << a))) continue;
    if (!b->physical[a][0] && !b->physical[a][1]) continue;
    ax.axis[na] = a;
    ax.lo[na] = b->physical[a][0];
    ax.hi[na] = b->physical[a][1];
    ++na;
    work = std::max(work, 2LL * layers * b->n[(a + 1) % 3] * b->n[(a + 2) % 3]);
  }
  if (na == 0) return 0;
  if (work >= (1LL << 31)) {
    set_error("apply_boundaries: face slab too large for one launch");
    return PPMLR_INVALID_SPEC;
  }
  bc_kernel<<<dim3(grid_for(work), na), 256, 0, b->stream>>>(s, L, ax, layers, b->boundary);
  b->kernel_launches += 1;
  CK(cudaGetLastError());
  return 0;
}

int launch_cfl(ppmlr_gpu_block* b, unsigned long long step_add) {
  const Lay L = lay_of(b);
  Planes s = planes(cur_buf(b), b->fs);
  const long long work = (long long)b->n[0] * b->n[1] * b->n[2];
  const double* bd0 = b->bd ? b->bd : nullptr;
  const double* bd1 = b->bd ? b->bd + b->fs : nullptr;
  const double* bd2 = b->bd ? b->bd + 2 * b->fs : nullptr;
  if (b->with_dipole)
    cfl_kernel<true><<<grid_for(work), 256, 0, b->stream>>>(s, L, bd0, bd1, bd2, b->ax[0].dx,
                                                             b->ax[1].dx, b->ax[2].dx, b->c,
                                                             ctx_of(b), step_add);
  else
    cfl_kernel<false><<<grid_for(work), 256, 0, b->stream>>>(s, L, bd0, bd1, bd2, b->ax[0].dx,
                                                              b->ax[1].dx, b->ax[2].dx, b->c,
                                                              ctx_of(b), step_add);
  CK(cudaGetLastError());
  b->kernel_launches += 1;
  return 0;
}

int launch_sources(ppmlr_gpu_block* b, int fuse_cfl, int part) {
  SrcArgs A;
  const int src = part == 2 ? b->cur ^ 1 : b->cur;  // as launch_sweep
  A.in = planes(b->buf[src], b->fs);
  A.out = planes(b->buf[src ^ 1], b->fs);
  A.L = lay_of(b);
  A.bd0 = b->bd ? b->bd : nullptr;
  A.bd1 = b->bd ? b->bd + b->fs : nullptr;
  A.bd2 = b->bd ? b->bd + 2 * b->fs : nullptr;
  A.hm0 = b->ax[0].hm;
  A.hp0 = b->ax[0].hp;
  A.hm1 = b->ax[1].hm;
  A.hp1 = b->ax[1].hp;
  A.hm2 = b->ax[2].hm;
  A.hp2 = b->ax[2].hp;
  A.den0 = b->ax[0].den;
  A.den1 = b->ax[1].den;
  A.den2 = b->ax[2].den;
  A.rden0 = b->ax[0].rden;
  A.rden1 = b->ax[1].rden;
  A.rden2 = b->ax[2].rden;
  A.dx0 = b->ax[0].dx;
  A.dx1 = b->ax[1].dx;
  A.dx2 = b->ax[2].dx;
  A.fl0 = b->fbox_lo[0];
  A.fl1 = b->fbox_lo[1];
  A.fl2 = b->fbox_lo[2];
  A.fn0 = b->fbox_n[0];
  A.fn1 = b->fbox_n[1];
  A.fn2 = b->fbox_n[2];
  A.fslot = b->fslot;
  A.fst = b->fstates;
  A.nfrozen = b->n_frozen;
  A.c = b->c;
  A.ctx = ctx_of(b);
  A.fuse_cfl = fuse_cfl;
  A.redo_count = b->d_redo;
  A.redo_list = b->d_redo + 1;
  A.redo_cap = b->redo_cap;
  A.part = part;
  split_range(b->n[0], PPMLR_KNS::kSrcTX, (b->n[0] + PPMLR_KNS::kSrcTX - 1) / PPMLR_KNS::kSrcTX,
              A.cl, A.cr);
  CK(cudaMemsetAsync(b->d_redo, 0, sizeof(unsigned), b->stream));
  const cudaError_t e = b->precision == PPMLR_FAST
                            ? launch_sources_fast(A, b->src_maps[src], b->with_dipole,
                                                  b->stream)
                            : launch_sources_strict(A, b->src_maps[src], b->with_dipole,
                                                    b->stream);
  if (e != cudaSuccess) return cuda_fail(e, "sources kernel launch");
  b->kernel_launches += 2;
  if (part != 2) b->cur ^= 1;
  return 0;
}

int launch_frozen(ppmlr_gpu_block* b) {
  if (b->n_frozen <= 0) return 0;
  frozen_restore_kernel<<<grid_for(b->n_frozen), 256, 0, b->stream>>>(
      planes(cur_buf(b), b->fs), b->fidx, b->fstates, b->n_frozen);
  CK(cudaGetLastError());
  b->kernel_launches += 1;
  return 0;
}

int launch_step_end(ppmlr_gpu_block* b, double cfl, int close_step, int have_min) {
  step_end_kernel<<<1, 1, 0, b->stream>>>(ctx_of(b), cfl, close_step, have_min);
  CK(cudaGetLastError());
  b->kernel_launches += 1;
  return 0;
}

}  // namespace ppmlr_b200

namespace ppmlr_b200 {
int block_set_dt(ppmlr_gpu_block* b, double dt) {
  b->dt_valid = false;  // state or dt slot changes
  if (dt < 0.0) return 0;  // use the device slot as is
  b->h_pinned[1] = dt;
  CK(cudaMemcpyAsync(b->d_dt, &b->h_pinned[1], 8, cudaMemcpyHostToDevice, b->stream));
  return 0;
}
}  // namespace ppmlr_b200

// ---------------------------------------------------------------- C-ABI

#ifndef PPMLR_TMA_L2_PROMOTION
#define PPMLR_TMA_L2_PROMOTION CU_TENSOR_MAP_L2_PROMOTION_L2_256B  // measured +0.5-0.8%
#endif

namespace {
// TMA descriptors of the sweep inputs for both ping-pong buffers and every
// axis: each field / dipole plane as a 3-D tensor {S0, S1, S2} (x pitch P0)
// with the axis' tile box (sweep.cuh SweepMaps).  cuTensorMapEncodeTiled is
// reached through the runtime's driver entry point (no -lcuda).
int build_sweep_maps(ppmlr_gpu_block* b) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return PPMLR_RUNTIME;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  b->maps = new SweepMaps[6];
  std::memset(static_cast<void*>(b->maps), 0, sizeof(SweepMaps) * 6);
  b->src_maps = new SrcMaps[2];
  std::memset(static_cast<void*>(b->src_maps), 0, sizeof(SrcMaps) * 2);
  const cuuint32_t l0 = b->sweep_L[0], l1 = b->sweep_L[1], l2 = b->sweep_L[2];
  const cuuint32_t np = kSweepNP;
  const cuuint32_t obox[3][3] = {{l0, np, 1}, {np, l1, 1}, {np, 1, l2}};
  const cuuint64_t dims[3] = {(cuuint64_t)b->S[0], (cuuint64_t)b->S[1], (cuuint64_t)b->S[2]};
  const cuuint64_t strides[2] = {(cuuint64_t)b->sy * 8, (cuuint64_t)b->sz * 8};
  const cuuint32_t elem[3] = {1, 1, 1};
  // tile box per axis: TL = L + 8 strip positions x 4 pencils
  const cuuint32_t t0 = b->sweep_L[0] + 8, t1 = b->sweep_L[1] + 8, t2 = b->sweep_L[2] + 8;
  const cuuint32_t box[3][3] = {{t0, np, 1}, {np, t1, 1}, {np, 1, t2}};
  for (int k = 0; k < 2; ++k)
    for (int a = 0; a < 3; ++a) {
      SweepMaps& m = b->maps[3 * k + a];
      for (int f = 0; f < 11; ++f) {
        if (f >= 8 && !b->bd) break;
        double* base = f < 8 ? b->buf[k] + f * b->fs : b->bd + (f - 8) * b->fs;
        CUtensorMap* t = f < 8 ? &m.f[f] : &m.bd[f - 8];
        const CUresult r = encode(t, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides,
                                  box[a], elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  CU_TENSOR_MAP_SWIZZLE_NONE, PPMLR_TMA_L2_PROMOTION,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
          set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
          return PPMLR_RUNTIME;
        }
      }
      if (a == 0) {  // the source kernel's plane boxes (v, B', dipole)
        SrcMaps& sm = b->src_maps[k];
        const cuuint32_t pbox[3] = {(cuuint32_t)PPMLR_KNS::kSrcHX, (cuuint32_t)PPMLR_KNS::kSrcHY, 1};
        for (int f = 0; f < 9; ++f) {
          if (f >= 6 && !b->bd) break;
          double* base = f < 6 ? b->buf[k] + (1 + f) * b->fs : b->bd + (f - 6) * b->fs;
          const CUresult r = encode(&sm.f[f], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims,
                                    strides, pbox, elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    CU_TENSOR_MAP_SWIZZLE_NONE,
                                    PPMLR_TMA_L2_PROMOTION,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          if (r != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
            return PPMLR_RUNTIME;
          }
        }
      }
      for (int f = 0; f < 8; ++f) {  // results go to the other buffer
        const CUresult r = encode(&m.out[f], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                                  b->buf[k ^ 1] + f * b->fs, dims, strides, obox[a], elem,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
          set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
          return PPMLR_RUNTIME;
        }
      }
    }
  return 0;
}
}  // namespace

extern "C" {

const char* ppmlr_gpu_last_error(void) { return g_last_error.c_str(); }

const char* ppmlr_gpu_version(void) {
  return "ppmlr-b200 0.1 (sm_100a, FP64 PPMLR sweeps; strict+fast)";
}

int ppmlr_gpu_block_create(const ppmlr_gpu_block_desc* d, ppmlr_gpu_block** out) {
  *out = nullptr;
  if (!d) {
    set_error("null descriptor");
    return PPMLR_INVALID_SPEC;
  }
  for (int a = 0; a < 3; ++a)
    if (d->n[a] < 1) {
      set_error("block dimensions must be positive");
      return PPMLR_INVALID_SPEC;
    }
  if (d->ghost < 4) {
    set_error("ghost width must be >= 4");
    return PPMLR_INVALID_SPEC;
  }
  // the first-failure error keys (ppmlr_common.hpp) address strip positions
  // in 17 bits and the pencils of a face in 27
  for (int a = 0; a < 3; ++a)
    if (d->n[a] + 2 * kG >= kMaxStrip ||
        (unsigned long long)d->n[(a + 1) % 3] * d->n[(a + 2) % 3] >= kMaxPencils) {
      set_error("block too large for the error-key fields: an axis must have fewer than "
                "131064 cells and a face fewer than 2^27 pencils");
      return PPMLR_INVALID_SPEC;
    }
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (d->device < 0 || d->device >= ndev) {
    set_error("no such CUDA device");
    return PPMLR_RUNTIME;
  }
  CK(cudaSetDevice(d->device));
  auto* b = new ppmlr_gpu_block();
  b->device = d->device;
  b->g_ref = d->ghost;
  for (int a = 0; a < 3; ++a) {
    b->n[a] = d->n[a];
    b->lo[a] = d->lo[a];
    b->S[a] = d->n[a] + 2 * kG;
    b->physical[a][0] = d->physical[a][0];
    b->physical[a][1] = d->physical[a][1];
  }
  b->c.gamma = d->gamma;
  b->c.mu0 = d->mu0;
  b->c.pressure_floor = d->pressure_floor;
  b->c.gm1 = d->gamma - 1.0;
  b->c.two_mu0 = 2.0 * d->mu0;
  b->boundary = d->boundary;
  b->wind[0] = d->wind_rho;
  b->wind[1] = d->wind_v[0];
  b->wind[2] = d->wind_v[1];
  b->wind[3] = d->wind_v[2];
  b->wind[4] = d->wind_imf[0];
  b->wind[5] = d->wind_imf[1];
  b->wind[6] = d->wind_imf[2];
  b->wind[7] = d->wind_p;
  b->with_dipole = d->with_dipole != 0;
  b->precision = d->precision;
  set_state_layout(b);
  if (d->boundary == PPMLR_BC_PERIODIC)
    for (int a = 0; a < 3; ++a)
      if (b->physical[a][0] != b->physical[a][1] || (b->physical[a][0] && b->n[a] < d->ghost)) {
        b->deferred_error = "periodic boundaries need whole-axis blocks";
        b->deferred_code = PPMLR_INVALID_SPEC;
      }
  auto fail = [&](int rc) {
    ppmlr_gpu_block_destroy(b);
    return rc;
  };
  int rc = 0;
  // geometry windows and tables
  for (int a = 0; a < 3; ++a) {
    const int off = d->ghost - kG;
    const int span = b->S[a];
    b->h_centers[a].assign(d->centers[a] + off, d->centers[a] + off + span);
    b->h_spacings[a].assign(d->spacings[a] + off, d->spacings[a] + off + span);
    std::vector<double> slope, qfc, hm, hp;
    build_axis_tables(b->h_spacings[a], b->h_centers[a], slope, qfc, hm, hp);
    if (b->precision == PPMLR_FAST) {
      // fast build: folded factors (ppmlr_dev.cuh kSlopeN / kQfcN)
      std::vector<double> s2(2 * span), q3(3 * (span + 1));
      for (int l = 0; l < span; ++l) {
        s2[2 * l] = slope[3 * l] * slope[3 * l + 1];
        s2[2 * l + 1] = slope[3 * l] * slope[3 * l + 2];
      }
      for (int m = 0; m <= span; ++m) {
        const double* e = &qfc[5 * m];
        q3[3 * m] = e[0] + e[1] * e[2];
        q3[3 * m + 1] = -(e[1] * e[3]);
        q3[3 * m + 2] = e[1] * e[4];
      }
      slope.swap(s2);
      qfc.swap(q3);
    }
    b->ax[a].span = span;
    if ((rc = upload_vec(&b->ax[a].dx, b->h_spacings[a]))) return fail(rc);
    if ((rc = upload_vec(&b->ax[a].slope, slope))) return fail(rc);
    if ((rc = upload_vec(&b->ax[a].qfc, qfc))) return fail(rc);
    if ((rc = upload_vec(&b->ax[a].hm, hm))) return fail(rc);
    if ((rc = upload_vec(&b->ax[a].hp, hp))) return fail(rc);
    std::vector<double> den(span, 1.0);
    for (int l = 1; l + 1 < span; ++l) den[l] = (hm[l] * hp[l]) * (hm[l] + hp[l]);
    if ((rc = upload_vec(&b->ax[a].den, den))) return fail(rc);
    if ((rc = upload_vec(&b->ax[a].rdx, b->h_spacings[a]))) return fail(rc);
    if ((rc = upload_vec(&b->ax[a].rden, den))) return fail(rc);
    rcp_table_kernel<<<(span + 127) / 128, 128>>>(b->ax[a].rdx, span);
    rcp_table_kernel<<<(span + 127) / 128, 128>>>(b->ax[a].rden, span);
    if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
      set_error("rcp_table_kernel failed");
      return fail(PPMLR_RUNTIME);
    }
  }
  {  // reciprocals of the run constants, refined on the device once
    std::vector<double> rc5 = {b->c.gm1, b->c.two_mu0, b->c.mu0, 6.0, 3.0};
    double* d5 = nullptr;
    if ((rc = upload_vec(&d5, rc5))) return fail(rc);
    rcp_table_kernel<<<1, 32>>>(d5, 5);
    const cudaError_t e5 = cudaMemcpy(rc5.data(), d5, 5 * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(d5);
    if (e5 != cudaSuccess) return fail(cuda_fail(e5, "constant reciprocals"));
    b->c.r_gm1 = rc5[0];
    b->c.r_two_mu0 = rc5[1];
    b->c.r_mu0 = rc5[2];
    b->c.r6 = rc5[3];
    b->c.r3 = rc5[4];
  }
  cudaError_t e;
  if ((e = cudaMalloc(&b->arena, sizeof(double) * b->ncell)) != cudaSuccess)
    return fail(cuda_fail(e, "cudaMalloc(state)"));
  if ((e = cudaMemset(b->arena, 0, sizeof(double) * b->ncell)) != cudaSuccess)
    return fail(cuda_fail(e, "cudaMemset(state)"));
  b->buf[0] = b->arena;
  b->buf[1] = b->arena + 8 * b->fs;
  if (b->with_dipole) b->bd = b->arena + 16 * b->fs;
  if (b->with_dipole) {  // y and z bricks: +2 x 3 x 8 B per cell (C5 +29 GB)
    b->bdz_ngx = (b->n[0] + 3) / 4;
    for (int a = 1; a < 3; ++a) {
      b->bdz_cs[a - 1] = (long long)b->n[a == 1 ? 2 : 1] * b->bdz_ngx * b->S[a] * 4;
      if ((e = cudaMalloc(&b->bdz[a - 1], sizeof(double) * 3 * b->bdz_cs[a - 1])) !=
          cudaSuccess)
        return fail(cuda_fail(e, "cudaMalloc(bd bricks)"));
      // consistent with the zeroed B_d planes until the first upload
      if ((e = cudaMemset(b->bdz[a - 1], 0, sizeof(double) * 3 * b->bdz_cs[a - 1])) !=
          cudaSuccess)
        return fail(cuda_fail(e, "cudaMemset(bd bricks)"));
    }
    b->bd_dirty = false;
  }
  if ((e = cudaMalloc(&b->d_err, 64)) != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc"));
  b->d_step = b->d_err + 1;
  b->d_min = b->d_err + 2;
  b->d_dt = reinterpret_cast<double*>(b->d_err + 3);
  b->d_dt_prev = reinterpret_cast<double*>(b->d_err + 4);
  b->d_time = reinterpret_cast<double*>(b->d_err + 5);
  {
    unsigned long long init[8] = {kNoError, 0, kInfBits, 0, 0, 0, 0, 0};
    cudaMemcpy(b->d_err, init, sizeof init, cudaMemcpyHostToDevice);
  }
  if ((e = cudaMallocHost(&b->h_pinned, 8 * sizeof(double))) != cudaSuccess)
    return fail(cuda_fail(e, "cudaMallocHost"));
  if ((e = cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking)) != cudaSuccess)
    return fail(cuda_fail(e, "cudaStreamCreate"));
  choose_sweep_tiles(b);
  if (int rc = build_sweep_maps(b)) return fail(rc);
  {
    long long tiles = 1;
    for (int a = 0; a < 3; ++a) {
      const int G = a == 0 ? 1 : 0, O = a == 2 ? 1 : 2;
      const long long t = (long long)((b->n[a] + b->sweep_L[a] - 1) / b->sweep_L[a]) *
                          ((b->n[G] + kSweepNP - 1) / kSweepNP) * b->n[O];
      tiles = std::max(tiles, t);
    }
    const long long cells = (long long)b->n[0] * b->n[1] * b->n[2];
    b->redo_cap = (unsigned)std::max<long long>(tiles, std::min<long long>(cells, 1 << 22));
    if ((e = cudaMalloc(&b->d_redo, sizeof(unsigned) * ((size_t)b->redo_cap + 2))) != cudaSuccess)
      return fail(cuda_fail(e, "cudaMalloc(redo)"));
  }
  *out = b;
  return 0;
}

void ppmlr_gpu_block_destroy(ppmlr_gpu_block* b) {
  if (!b) return;
  cudaSetDevice(b->device);
  if (b->stream) cudaStreamSynchronize(b->stream);
  for (auto& row : b->graphs)
    for (auto& g : row)
      if (g.exec) cudaGraphExecDestroy(g.exec);
  cudaFree(b->arena);
  cudaFree(b->bdz[0]);
  cudaFree(b->bdz[1]);
  for (int a = 0; a < 3; ++a) {
    cudaFree(b->ax[a].dx);
    cudaFree(b->ax[a].slope);
    cudaFree(b->ax[a].qfc);
    cudaFree(b->ax[a].hm);
    cudaFree(b->ax[a].hp);
    cudaFree(b->ax[a].rdx);
    cudaFree(b->ax[a].den);
    cudaFree(b->ax[a].rden);
  }
  delete[] b->maps;
  delete[] b->src_maps;
  if (b->snap_stream) cudaStreamSynchronize(b->snap_stream);
  cudaFree(b->d_snap);
  if (b->snap_stream) cudaStreamDestroy(b->snap_stream);
  if (b->copy_stream) cudaStreamDestroy(b->copy_stream);
  if (b->snap_ready) cudaEventDestroy(b->snap_ready);
  cudaFree(b->fslot);
  cudaFree(b->fstates);
  cudaFree(b->fidx);
  cudaFree(b->d_err);
  cudaFree(b->d_redo);
  cudaFree(b->d_scratch);
  if (b->h_pinned) cudaFreeHost(b->h_pinned);
  for (auto& ev : b->ev)
    if (ev) cudaEventDestroy(ev);
  for (auto ev : b->timing.pool) cudaEventDestroy(ev);
  if (b->stream && b->own_stream) cudaStreamDestroy(b->stream);
  delete b;
}

static int ensure_copy_stream(ppmlr_gpu_block* b) {
  if (!b->copy_stream) CK(cudaStreamCreateWithFlags(&b->copy_stream, cudaStreamNonBlocking));
  return 0;
}

static int ensure_scratch(ppmlr_gpu_block* b, size_t bytes) {
  if (b->scratch_bytes >= bytes) return 0;
  cudaFree(b->d_scratch);
  b->d_scratch = nullptr;
  CK(cudaMalloc(&b->d_scratch, bytes));
  b->scratch_bytes = bytes;
  return 0;
}

}  // extern "C"

namespace ppmlr_b200 {

// Frozen inner core (init_magnetosphere, stepper.cpp:107-110): bounding-box
// slot map + SoA states on the device; linear indices in the caller's
// (ghost g_ref) layout.
// Instantiated step graphs bake in kernel arguments (the frozen-core slot
// map's pointers and bounding box among them); anything that changes those
// must drop them so the next step re-captures.
static void drop_step_graphs(ppmlr_gpu_block* b) {
  for (auto& row : b->graphs)
    for (auto& g : row)
      if (g.exec) {
        cudaGraphExecDestroy(g.exec);
        g.exec = nullptr;
      }
}

int block_set_frozen(ppmlr_gpu_block* b, const int64_t* frozen_idx, const double* frozen_states,
                     int64_t n_frozen) {
  CK(cudaSetDevice(b->device));
  CK(cudaStreamSynchronize(b->stream));  // no step in flight reads the old map
  drop_step_graphs(b);
  const int gr = b->g_ref;
  const int S0r = b->n[0] + 2 * gr, S1r = b->n[1] + 2 * gr;
  const Lay L = lay_of(b);
  cudaFree(b->fslot);
  cudaFree(b->fstates);
  cudaFree(b->fidx);
  b->fslot = nullptr;
  b->fstates = nullptr;
  b->fidx = nullptr;
  b->n_frozen = n_frozen;
  if (n_frozen > 0) {
    int lo[3] = {1 << 30, 1 << 30, 1 << 30}, hi[3] = {-1, -1, -1};
    std::vector<int> ijk(3 * n_frozen);
    std::vector<long long> didx(n_frozen);
    for (int64_t f = 0; f < n_frozen; ++f) {
      const int64_t r = frozen_idx[f];
      const int i = (int)(r % S0r) - gr, j = (int)((r / S0r) % S1r) - gr,
                k = (int)(r / ((int64_t)S0r * S1r)) - gr;
      if (i < 0 || j < 0 || k < 0 || i >= b->n[0] || j >= b->n[1] || k >= b->n[2]) {
        set_error("frozen-core index outside the block interior");
        return PPMLR_INVALID_SPEC;
      }
      ijk[3 * f] = i;
      ijk[3 * f + 1] = j;
      ijk[3 * f + 2] = k;
      const int c3[3] = {i, j, k};
      for (int a = 0; a < 3; ++a) {
        lo[a] = std::min(lo[a], c3[a]);
        hi[a] = std::max(hi[a], c3[a]);
      }
      didx[f] = L.idx(i, j, k);
    }
    for (int a = 0; a < 3; ++a) {
      b->fbox_lo[a] = lo[a];
      b->fbox_n[a] = hi[a] - lo[a] + 1;
    }
    const size_t vol = (size_t)b->fbox_n[0] * b->fbox_n[1] * b->fbox_n[2];
    std::vector<int> slot(vol, -1);
    std::vector<double> st(8 * (size_t)n_frozen);
    for (int64_t f = 0; f < n_frozen; ++f) {
      const size_t v = (size_t)(ijk[3 * f] - lo[0]) +
                       b->fbox_n[0] * ((size_t)(ijk[3 * f + 1] - lo[1]) +
                                       b->fbox_n[1] * (size_t)(ijk[3 * f + 2] - lo[2]));
      slot[v] = (int)f;  // later entries win, like sequential restore
      for (int q = 0; q < 8; ++q) st[(size_t)q * n_frozen + f] = frozen_states[8 * f + q];
    }
    if (int rc = upload_vec(&b->fslot, slot)) return rc;
    if (int rc = upload_vec(&b->fstates, st)) return rc;
    if (int rc = upload_vec(&b->fidx, didx)) return rc;
  }
  return 0;
}

// Streamed upload: `fill(kr0, nk, fields, bd)` writes reference-layout AoS
// k-planes [kr0, kr0+nk) (bd only when the block carries the dipole) into
// pinned staging; each chunk is copied and converted while the next is
// filled.  No full-size host copy of the state is needed.
int block_upload_streamed(ppmlr_gpu_block* b, const ChunkFill& fill, bool with_bd,
                          const double* src_fields, const double* src_bd) {
  CK(cudaSetDevice(b->device));
  CK(cudaStreamSynchronize(b->stream));
  const int gr = b->g_ref;
  const int S0r = b->n[0] + 2 * gr, S1r = b->n[1] + 2 * gr, S2r = b->n[2] + 2 * gr;
  const size_t plane = (size_t)S0r * S1r;
  with_bd = with_bd && b->with_dipole && b->bd;
  if (with_bd) b->bd_dirty = true;
  const int nper = with_bd ? 11 : 8;
  const int kchunk = (int)std::max<size_t>(1, std::min<size_t>(S2r, (64ull << 20) / (plane * 8 * nper)));
  const size_t chunk_doubles = plane * kchunk * nper;
  if (int rc = ensure_scratch(b, 2 * chunk_doubles * sizeof(double))) return rc;
  // src_fields given: copy straight from the caller's buffers (pinned
  // memory DMAs at full PCIe rate); otherwise fill pinned staging chunks
  const bool direct = src_fields != nullptr;
  if (int rc = ensure_copy_stream(b)) return rc;
  // chunk copies on the copy stream, conversion kernels on the block stream:
  // the copy of chunk q+1 overlaps the kernels of chunk q (cdone: copy into
  // scratch q finished; kdone: kernels done with scratch q)
  struct Staging {  // released on every exit path (CK returns, a throwing fill)
    cudaStream_t st, cs;
    double* host[2] = {nullptr, nullptr};
    cudaEvent_t cdone[2] = {nullptr, nullptr}, kdone[2] = {nullptr, nullptr};
    ~Staging() {
      cudaStreamSynchronize(cs);
      cudaStreamSynchronize(st);
      for (int k = 0; k < 2; ++k) {
        if (host[k]) cudaFreeHost(host[k]);
        if (cdone[k]) cudaEventDestroy(cdone[k]);
        if (kdone[k]) cudaEventDestroy(kdone[k]);
      }
    }
  } stg{b->stream, b->copy_stream};
  double** host = stg.host;
  cudaEvent_t* cdone = stg.cdone;
  cudaEvent_t* kdone = stg.kdone;
  for (int q = 0; q < 2; ++q) {
    if (!direct) CK(cudaMallocHost(&host[q], chunk_doubles * sizeof(double)));
    CK(cudaEventCreateWithFlags(&cdone[q], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&kdone[q], cudaEventDisableTiming));
  }
  const cudaStream_t cs = b->copy_stream;
  const Lay L = lay_of(b);
  int rc = 0;
  int q = 0;
  for (int kr0 = 0; kr0 < S2r && !rc; kr0 += kchunk, q ^= 1) {
    const int nk = std::min(kchunk, S2r - kr0);
    double* dscr = b->d_scratch + q * chunk_doubles;
    const double* hb = nullptr;
    CK(cudaStreamWaitEvent(cs, kdone[q], 0));  // scratch q free again
    if (direct) {
      CK(cudaMemcpyAsync(dscr, src_fields + plane * kr0 * 8, plane * nk * 8 * sizeof(double),
                         cudaMemcpyHostToDevice, cs));
      if (with_bd) {
        CK(cudaMemcpyAsync(dscr + plane * nk * 8, src_bd + plane * kr0 * 3,
                           plane * nk * 3 * sizeof(double), cudaMemcpyHostToDevice, cs));
        hb = src_bd;
      }
    } else {
      CK(cudaEventSynchronize(cdone[q]));  // host staging q free again
      double* hf = host[q];
      double* hbw = with_bd ? host[q] + plane * nk * 8 : nullptr;
      fill(kr0, nk, hf, hbw);
      hb = hbw;
      CK(cudaMemcpyAsync(dscr, hf, plane * nk * nper * sizeof(double), cudaMemcpyHostToDevice,
                         cs));
    }
    CK(cudaEventRecord(cdone[q], cs));
    CK(cudaStreamWaitEvent(b->stream, cdone[q], 0));
    for (int k = 0; k < 2; ++k)
      aos_to_soa_kernel<<<grid_for(plane * nk), 256, 0, b->stream>>>(
          dscr, 8, planes(b->buf[k], b->fs), L, gr, S0r, S1r, kr0, nk,
          (k == 0 && hb) ? dscr + plane * nk * 8 : nullptr, b->bd,
          b->bd ? b->bd + b->fs : nullptr, b->bd ? b->bd + 2 * b->fs : nullptr);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaEventRecord(kdone[q], b->stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "streamed upload");
  }
  if (rc) return rc;
  CK(cudaStreamSynchronize(b->stream));
  return block_finish_upload(b);
}

// Pre-filled sunward shell, fresh error window and step counter.
// ---------------------------------------------------------------- multi-block
// Global dt of an in-process multi-block (multi-device) harness: every
// block's slot holds cfl * its local CFL min; one thread takes the min over
// all slots (peer loads when the blocks live on other GPUs) and writes it
// back to every slot.  min commutes with the monotone cfl * x, so this is
// compute_global_dt (harness.cpp:45-50) bit for bit.
__global__ void dt_min_all_kernel(double* const* slots, int n) {
  double m = *slots[0];
  for (int r = 1; r < n; ++r) m = fmin(m, *slots[r]);
  for (int r = 0; r < n; ++r) *slots[r] = m;
}

int launch_dt_min_all(double* const* d_slots, int n, cudaStream_t st) {
  dt_min_all_kernel<<<1, 1, 0, st>>>(d_slots, n);
  CK(cudaGetLastError());
  return 0;
}

int block_begin_window(ppmlr_gpu_block* b, long first_step) {
  CK(cudaSetDevice(b->device));
  unsigned long long init[2] = {kNoError, 0};
  CK(cudaMemcpyAsync(b->d_err, init, sizeof init, cudaMemcpyHostToDevice, b->stream));
  b->step_base = first_step;
  return 0;
}

int block_read_error(ppmlr_gpu_block* b, unsigned long long* key, unsigned long long* step) {
  CK(cudaSetDevice(b->device));
  CK(cudaMemcpyAsync(b->h_pinned + 4, b->d_err, 16, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  std::memcpy(key, b->h_pinned + 4, 8);
  std::memcpy(step, b->h_pinned + 5, 8);
  return 0;
}

int block_last_dt_time(ppmlr_gpu_block* b, double* dt, double* time) {
  CK(cudaSetDevice(b->device));
  CK(cudaMemcpyAsync(b->h_pinned + 2, b->d_dt_prev, 8, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(b->h_pinned + 3, b->d_time, 8, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  *dt = b->h_pinned[2];
  *time = b->h_pinned[3];
  return 0;
}

int block_reset_error(ppmlr_gpu_block* b) {
  CK(cudaSetDevice(b->device));
  const unsigned long long reset = kNoError;
  CK(cudaMemcpy(b->d_err, &reset, 8, cudaMemcpyHostToDevice));
  return 0;
}

int block_raise_error(ppmlr_gpu_block* b, unsigned long long key) {
  std::string msg;
  const int rc = decode_error(b, key, msg);
  set_error(msg);
  return rc;
}

// ---------------------------------------------------------------- device setup
// make_block's default state and dipole (stepper.cpp:63-69) and the built-in
// init_with ICs (harness.cpp:35-43; kinds 0 uniform, 1 Brio-Wu, 2
// Orszag-Tang, 3 blast) evaluated on the device, straight into the SoA
// buffers.  The expressions are the host restatement's (host.cpp make_ic /
// dipole) in the same IEEE operation order; this TU is compiled with
// --fmad=false and IEEE `/` and `sqrt`, so every value is bit-identical to
// the host path.  The one transcendental, Orszag-Tang's sin(), depends on a
// single coordinate: the host evaluates it per x / y centre (std::sin, as
// the reference) and the kernel reads those tables.
struct InitArgs {
  const double* cen[3];  // kG-ghost centre windows (S[a] entries)
  const double* tab;     // kind 2: sin(x_i) [S0], sin(2 x_i) [S0], sin(y_j) [S1]
  double p[8];
  int kind;
  double mu0;
};

__device__ __forceinline__ double dot3d(double ax, double ay, double az, double bx, double by,
                                        double bz) {
  return (ax * bx + ay * by) + az * bz;
}

__global__ void init_state_kernel(Planes d0, Planes d1, double* bd0, double* bd1, double* bd2,
                                  Lay L, int S0, int S1, int S2, InitArgs A, int* err) {
  const long long total = (long long)S0 * S1 * S2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int il = (int)(t % S0), jl = (int)((t / S0) % S1), kl = (int)(t / ((long long)S0 * S1));
    const double x = A.cen[0][il], y = A.cen[1][jl], z = A.cen[2][kl];
    double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    switch (A.kind) {
      case -2:  // make_block: {1, 0, 0, 1}
        s[0] = 1.0;
        s[7] = 1.0;
        break;
      case 0:
        for (int f = 0; f < 8; ++f) s[f] = A.p[f];
        break;
      case 1: {  // Brio-Wu
        const bool left = x < 0.5;
        s[0] = left ? 1.0 : 0.125;
        s[7] = left ? 1.0 : 0.1;
        s[4] = 0.75;
        s[5] = left ? 1.0 : -1.0;
        s[6] = 0.0;
        break;
      }
      case 2: {  // Orszag-Tang
        const double g = A.p[0];
        const double sx = A.tab[il], s2x = A.tab[S0 + il], sy = A.tab[2 * S0 + jl];
        s[0] = g * g;
        s[7] = g;
        s[1] = -sy;
        s[2] = sx;
        s[3] = 0.0;
        s[4] = -sy;
        s[5] = s2x;
        s[6] = 0.0;
        break;
      }
      case 3: {  // blast per unit block
        const double cx = floor(x + 0.5);
        const double dx = x - cx;
        const double r2 = (dx * dx + y * y) + z * z;
        s[0] = 1.0;
        s[7] = r2 < A.p[2] * A.p[2] ? A.p[0] : A.p[1];
        s[4] = sqrt(0.5);
        s[5] = sqrt(0.5);
        break;
      }
    }
    const long long d = L.idx(il - kG, jl - kG, kl - kG);
#pragma unroll
    for (int f = 0; f < 8; ++f) {
      d0.f[f][d] = s[f];
      d1.f[f][d] = s[f];
    }
    if (bd0) {  // physics.cpp:14-21 dipole_field, moment (0, 0, -4 pi)
      const double kPiD = 3.14159265358979323846;
      const double mx = 0.0, my = 0.0, mz = -4.0 * kPiD;
      const double r2 = dot3d(x, y, z, x, y, z);
      if (r2 == 0.0) {
        atomicOr(err, 1);
        continue;
      }
      const double r = sqrt(r2);
      const double rx = x / r, ry = y / r, rz = z / r;
      const double k = A.mu0 / (4.0 * kPiD);
      const double sm = 3.0 * dot3d(mx, my, mz, rx, ry, rz);
      const double vx = rx * sm - mx, vy = ry * sm - my, vz = rz * sm - mz;
      const double den = r2 * r;
      bd0[d] = (vx * k) / den;
      bd1[d] = (vy * k) / den;
      bd2[d] = (vz * k) / den;
    }
  }
}

bool device_init_supported(int kind) { return kind >= -2 && kind <= 3 && kind != -1; }

int block_init_device(ppmlr_gpu_block* b, int kind, const double* params, bool with_bd) {
  CK(cudaSetDevice(b->device));
  CK(cudaStreamSynchronize(b->stream));
  with_bd = with_bd && b->with_dipole && b->bd;
  if (with_bd) b->bd_dirty = true;
  InitArgs A{};
  A.kind = kind;
  A.mu0 = b->c.mu0;
  if (params)
    for (int f = 0; f < 8; ++f) A.p[f] = params[f];
  std::vector<double> tab;
  size_t ncen = 0;
  for (int a = 0; a < 3; ++a) ncen += b->S[a];
  if (kind == 2) {
    tab.resize(2 * (size_t)b->S[0] + b->S[1]);
    for (int i = 0; i < b->S[0]; ++i) {
      tab[i] = std::sin(b->h_centers[0][i]);
      tab[b->S[0] + i] = std::sin(2.0 * b->h_centers[0][i]);
    }
    for (int j = 0; j < b->S[1]; ++j) tab[2 * b->S[0] + j] = std::sin(b->h_centers[1][j]);
  }
  const size_t need = sizeof(double) * (ncen + tab.size()) + sizeof(int);
  if (int rc = ensure_scratch(b, need)) return rc;
  std::vector<double> host(ncen + tab.size());
  size_t off = 0;
  for (int a = 0; a < 3; ++a) {
    std::copy(b->h_centers[a].begin(), b->h_centers[a].end(), host.begin() + off);
    A.cen[a] = b->d_scratch + off;
    off += b->S[a];
  }
  std::copy(tab.begin(), tab.end(), host.begin() + off);
  A.tab = b->d_scratch + off;
  int* d_err = reinterpret_cast<int*>(b->d_scratch + host.size());
  CK(cudaMemcpyAsync(b->d_scratch, host.data(), sizeof(double) * host.size(),
                     cudaMemcpyHostToDevice, b->stream));
  CK(cudaMemsetAsync(d_err, 0, sizeof(int), b->stream));
  const long long total = (long long)b->S[0] * b->S[1] * b->S[2];
  init_state_kernel<<<grid_for(total), 256, 0, b->stream>>>(
      planes(b->buf[0], b->fs), planes(b->buf[1], b->fs), with_bd ? b->bd : nullptr,
      with_bd ? b->bd + b->fs : nullptr, with_bd ? b->bd + 2 * b->fs : nullptr, lay_of(b),
      b->S[0], b->S[1], b->S[2], A, d_err);
  CK(cudaGetLastError());
  int herr = 0;
  CK(cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  if (herr) {
    set_error("dipole_field evaluated at the singularity");
    return PPMLR_UNPHYSICAL;
  }
  return block_finish_upload(b);
}

int block_finish_upload(ppmlr_gpu_block* b) {
  b->dt_valid = false;  // state or dt slot changes
  const Lay L = lay_of(b);
  if (b->bd_dirty) {
    for (int a = 1; a < 3; ++a)
      if (b->bdz[a - 1]) {
        bd_bricks_kernel<<<grid_for(3 * b->bdz_cs[a - 1]), 256, 0, b->stream>>>(
            b->bdz[a - 1], b->bd, b->fs, L, a, b->bdz_ngx, b->S[a], b->bdz_cs[a - 1]);
        CK(cudaGetLastError());
      }
    b->bd_dirty = false;
  }
  // Magnetosphere: constant sunward shell in both buffers.
  if (b->boundary == PPMLR_BC_MAGNETOSPHERE && b->physical[0][1]) {
    for (int k = 0; k < 2; ++k)
      wind_fill_kernel<<<grid_for((long long)kG * b->n[1] * b->n[2]), 256, 0, b->stream>>>(
          planes(b->buf[k], b->fs), L, b->bd, b->bd ? b->bd + b->fs : nullptr,
          b->bd ? b->bd + 2 * b->fs : nullptr, b->wind[0], b->wind[7], b->wind[1],
          b->wind[2], b->wind[3], b->wind[4], b->wind[5], b->wind[6]);
    CK(cudaGetLastError());
  }
  b->cur = 0;
  {
    unsigned long long init[6] = {kNoError, 0, kInfBits, 0, 0, 0};
    CK(cudaMemcpyAsync(b->d_err, init, sizeof init, cudaMemcpyHostToDevice, b->stream));
  }
  b->step_base = 0;
  CK(cudaStreamSynchronize(b->stream));
  return 0;
}

}  // namespace ppmlr_b200

extern "C" {

int ppmlr_gpu_block_upload(ppmlr_gpu_block* b, const double* fields, const double* bd,
                           const int64_t* frozen_idx, const double* frozen_states,
                           int64_t n_frozen) {
  const bool with_bd = b->with_dipole && bd != nullptr;
  if (int rc = block_set_frozen(b, frozen_idx, frozen_states, n_frozen)) return rc;
  return block_upload_streamed(b, ChunkFill(), with_bd, fields, bd);
}

static int download_impl(ppmlr_gpu_block* b, double* fields, bool interior_only) {
  CK(cudaSetDevice(b->device));
  const Lay L = lay_of(b);
  if (interior_only) {  // k-chunks through two 64 MB scratch halves
    const size_t plane = (size_t)b->n[0] * b->n[1];
    const int kchunk = (int)std::max<size_t>(1, std::min<size_t>(b->n[2], (64ull << 20) / (plane * 64)));
    const size_t half = plane * kchunk * 8;
    if (int rc = ensure_scratch(b, 2 * half * sizeof(double))) return rc;
    if (int rc = ensure_copy_stream(b)) return rc;
    // conversion kernels on the block stream, D2H copies on the copy stream
    // (the copy of chunk q overlaps the kernel of chunk q+1)
    struct Ev {
      cudaEvent_t e[4] = {nullptr, nullptr, nullptr, nullptr};
      ~Ev() {
        for (auto x : e)
          if (x) cudaEventDestroy(x);
      }
    } ev;
    for (auto& x : ev.e) CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    cudaEvent_t* kdone = ev.e;      // kernel wrote scratch q
    cudaEvent_t* cdone = ev.e + 2;  // copy read scratch q
    const cudaStream_t cs = b->copy_stream;
    CK(cudaEventRecord(cdone[0], cs));
    CK(cudaEventRecord(cdone[1], cs));
    int q = 0;
    for (int k0 = 0; k0 < b->n[2]; k0 += kchunk, q ^= 1) {
      const int nk = std::min(kchunk, b->n[2] - k0);
      double* dscr = b->d_scratch + q * half;
      CK(cudaStreamWaitEvent(b->stream, cdone[q], 0));
      soa_to_interior_kernel<<<grid_for(plane * nk), 256, 0, b->stream>>>(
          dscr, planes(cur_buf(b), b->fs), L, k0, nk);
      CK(cudaGetLastError());
      CK(cudaEventRecord(kdone[q], b->stream));
      CK(cudaStreamWaitEvent(cs, kdone[q], 0));
      CK(cudaMemcpyAsync(fields + plane * k0 * 8, dscr, plane * nk * 64, cudaMemcpyDeviceToHost,
                         cs));
      CK(cudaEventRecord(cdone[q], cs));
    }
    CK(cudaStreamSynchronize(cs));
    CK(cudaStreamSynchronize(b->stream));
    return 0;
  }
  const int gr = b->g_ref;
  const int S0r = b->n[0] + 2 * gr, S1r = b->n[1] + 2 * gr, S2r = b->n[2] + 2 * gr;
  const size_t plane = (size_t)S0r * S1r;
  const int kchunk = (int)std::max<size_t>(1, std::min<size_t>(S2r, (64ull << 20) / (plane * 64)));
  if (int rc = ensure_scratch(b, plane * kchunk * 64)) return rc;
  for (int kr0 = 0; kr0 < S2r; kr0 += kchunk) {
    const int nk = std::min(kchunk, S2r - kr0);
    soa_to_aos_kernel<<<grid_for(plane * nk), 256, 0, b->stream>>>(
        b->d_scratch, planes(cur_buf(b), b->fs), L, gr, S0r, S1r, kr0, nk);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(fields + plane * kr0 * 8, b->d_scratch, plane * nk * 64,
                       cudaMemcpyDeviceToHost, b->stream));
    CK(cudaStreamSynchronize(b->stream));
  }
  return 0;
}

int ppmlr_gpu_block_download(ppmlr_gpu_block* b, double* fields) {
  return download_impl(b, fields, false);
}
int ppmlr_gpu_block_download_interior(ppmlr_gpu_block* b, double* out) {
  return download_impl(b, out, true);
}

int ppmlr_gpu_block_snapshot_capture(ppmlr_gpu_block* b) {
  CK(cudaSetDevice(b->device));
  const long long cells = (long long)b->n[0] * b->n[1] * b->n[2];
  if (!b->snap_stream) {
    CK(cudaStreamCreateWithFlags(&b->snap_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&b->snap_ready, cudaEventDisableTiming));
  }
  // the previous capture must be fully drained before it is overwritten
  CK(cudaStreamSynchronize(b->snap_stream));
  if (!b->d_snap) CK(cudaMalloc(&b->d_snap, sizeof(double) * 8 * (size_t)cells));
  interior_planes_kernel<<<grid_for(cells), 256, 0, b->stream>>>(
      b->d_snap, planes(cur_buf(b), b->fs), lay_of(b));
  CK(cudaGetLastError());
  b->kernel_launches += 1;
  CK(cudaEventRecord(b->snap_ready, b->stream));
  return 0;
}

int ppmlr_gpu_block_snapshot_read(ppmlr_gpu_block* b, int field, int k0, int nk, double* dst,
                                  int64_t dst_pitch, int64_t dst_slice) {
  CK(cudaSetDevice(b->device));
  if (!b->d_snap || field < 0 || field > 7 || k0 < 0 || nk < 0 || k0 + nk > b->n[2] ||
      dst_pitch < b->n[0] || dst_slice < dst_pitch * b->n[1]) {
    set_error("snapshot_read: no capture or range outside the block interior");
    return PPMLR_INVALID_SPEC;
  }
  const size_t plane = (size_t)b->n[0] * b->n[1];
  const double* src = b->d_snap + (size_t)field * plane * b->n[2];
  CK(cudaStreamWaitEvent(b->snap_stream, b->snap_ready, 0));
  for (int k = 0; k < nk; ++k)
    CK(cudaMemcpy2DAsync(dst + (size_t)k * dst_slice, sizeof(double) * dst_pitch,
                         src + (size_t)(k0 + k) * plane, sizeof(double) * b->n[0],
                         sizeof(double) * b->n[0], b->n[1], cudaMemcpyDeviceToHost,
                         b->snap_stream));
  CK(cudaStreamSynchronize(b->snap_stream));
  return 0;
}

// defer_next_cfl: a non-finite CFL candidate that the fused pass found for
// the step after the window belongs to the next advance (the reference
// raises it from compute_global_dt at the top of that step): keep it out of
// this result and let the next run's standalone CFL pass raise it.
static int check_impl(ppmlr_gpu_block* b, bool defer_next_cfl) {
  CK(cudaSetDevice(b->device));
  CK(cudaMemcpyAsync(b->h_pinned + 4, b->d_err, 16, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  unsigned long long key, step;
  std::memcpy(&key, b->h_pinned + 4, 8);
  std::memcpy(&step, b->h_pinned + 5, 8);
  if (key == kNoError) return 0;
  b->dt_valid = false;
  if (defer_next_cfl && err_phase(key) == kPhaseCfl && err_step(key) == (step & kErrStepMask)) {
    const unsigned long long reset = kNoError;
    cudaMemcpy(b->d_err, &reset, 8, cudaMemcpyHostToDevice);
    return 0;
  }
  std::string msg;
  const int rc = decode_error(b, key, msg);
  set_error(msg);
  const unsigned long long reset = kNoError;
  cudaMemcpy(b->d_err, &reset, 8, cudaMemcpyHostToDevice);
  return rc;
}

int ppmlr_gpu_block_check(ppmlr_gpu_block* b) { return check_impl(b, false); }

static int deferred(ppmlr_gpu_block* b) {
  if (b->deferred_code) {
    set_error(b->deferred_error);
    return b->deferred_code;
  }
  return 0;
}

int ppmlr_gpu_block_compute_dt(ppmlr_gpu_block* b, double cfl, double* dt_out) {
  b->dt_valid = false;  // state or dt slot changes
  CK(cudaSetDevice(b->device));
  if (int rc = launch_cfl(b, 0)) return rc;
  if (int rc = launch_step_end(b, cfl, 0, 1)) return rc;
  CK(cudaMemcpyAsync(b->h_pinned + 6, b->d_dt, 8, cudaMemcpyDeviceToHost, b->stream));
  if (int rc = ppmlr_gpu_block_check(b)) return rc;  // uses h_pinned[4..5]
  *dt_out = b->h_pinned[6];
  return 0;
}

int ppmlr_gpu_block_local_dt_async(ppmlr_gpu_block* b, double cfl) {
  b->dt_valid = false;  // state or dt slot changes
  CK(cudaSetDevice(b->device));
  if (int rc = launch_cfl(b, 0)) return rc;
  return launch_step_end(b, cfl, 0, 1);
}

double* ppmlr_gpu_block_dt_slot(ppmlr_gpu_block* b) { return b->d_dt; }


int ppmlr_gpu_block_fill_boundaries(ppmlr_gpu_block* b, int axis_mask, int layers) {
  if (int rc = deferred(b)) return rc;
  CK(cudaSetDevice(b->device));
  if (layers < 1 || layers > kG) {
    set_error("fill_boundaries: layers must be in 1..4");
    return PPMLR_INVALID_SPEC;
  }
  return launch_bc(b, axis_mask, layers);
}

int ppmlr_gpu_block_sweep(ppmlr_gpu_block* b, int axis, double dt) {
  b->dt_valid = false;  // state or dt slot changes
  CK(cudaSetDevice(b->device));
  if (axis < 0 || axis > 2) {
    set_error("sweep: axis must be 0, 1 or 2");
    return PPMLR_INVALID_SPEC;
  }
  if (int rc = block_set_dt(b, dt)) return rc;
  // The sweep writes only interior cells of the other buffer; carry the
  // untouched cells (ghosts) over so the block behaves in place.
  CK(copy_state(b, b->buf[b->cur ^ 1], b->buf[b->cur]));
  if (int rc = launch_sweep(b, axis, kPhaseSweep0 + axis)) return rc;
  return 0;
}

int ppmlr_gpu_block_sources(ppmlr_gpu_block* b, double dt) {
  b->dt_valid = false;  // state or dt slot changes
  CK(cudaSetDevice(b->device));
  if (int rc = block_set_dt(b, dt)) return rc;
  CK(copy_state(b, b->buf[b->cur ^ 1], b->buf[b->cur]));
  // standalone apply_sources: no frozen override, no fused CFL
  const long long nf = b->n_frozen;
  b->n_frozen = 0;
  const int rc = launch_sources(b, 0);
  b->n_frozen = nf;
  return rc;
}

int ppmlr_gpu_block_restore_frozen(ppmlr_gpu_block* b) {
  b->dt_valid = false;  // state or dt slot changes
  CK(cudaSetDevice(b->device));
  return launch_frozen(b);
}

// One full step of a whole-domain block, stream-ordered, dt already in d_dt.
// A sweep launch bracketed by CUDA events when timing is on (the dominant
// kernel's in-run duration for bench.py's roofline).
static int timed_sweep(ppmlr_gpu_block* b, int axis, int phase, int part = 0) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (b->timing.enabled) {
    auto& t = b->timing;
    while (t.pool.size() < t.used + 2) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      t.pool.push_back(e);
    }
    e0 = t.pool[t.used];
    e1 = t.pool[t.used + 1];
    t.used += 2;
    CK(cudaEventRecord(e0, b->stream));
  }
  if (int rc = launch_sweep(b, axis, phase, part)) return rc;
  if (e1) CK(cudaEventRecord(e1, b->stream));
  return 0;
}

static int enqueue_step(ppmlr_gpu_block* b, double cfl, int with_sources, int parity) {
  static const int order[2][3] = {{0, 1, 2}, {2, 1, 0}};
  for (int s = 0; s < 3; ++s) {
    const int axis = order[parity][s];
    if (int rc = launch_bc(b, 1 << axis, kG)) return rc;
    if (int rc = timed_sweep(b, axis, kPhaseSweep0 + s)) return rc;
  }
  if (with_sources) {
    if (int rc = launch_bc(b, 7, 1)) return rc;
    if (int rc = launch_sources(b, 1)) return rc;
  } else {
    if (int rc = launch_frozen(b)) return rc;
    if (int rc = launch_cfl(b, 1)) return rc;
  }
  return launch_step_end(b, cfl, 1, 1);
}

static int run_steps(ppmlr_gpu_block* b, double cfl, int with_sources, long first_step,
                     long steps) {
  if (int rc = deferred(b)) return rc;
  CK(cudaSetDevice(b->device));
  // fresh error window; keys count steps from first_step
  {
    unsigned long long init[2] = {kNoError, 0};
    CK(cudaMemcpyAsync(b->d_err, init, sizeof init, cudaMemcpyHostToDevice, b->stream));
    b->step_base = first_step;
  }
  // dt of the first step, unless the previous run left it for this state
  if (!(b->dt_valid && b->dt_cfl == cfl)) {
    if (int rc = launch_cfl(b, 0)) return rc;
    if (int rc = launch_step_end(b, cfl, 0, 1)) return rc;
  }
  b->dt_valid = false;
  const bool use_graph = !b->timing.enabled && env_int("PPMLR_NO_GRAPH", 0) == 0;
  for (long s = 0; s < steps; ++s) {
    const int parity = (first_step + s) % 2 == 0 ? 0 : 1;
    if (!use_graph) {
      if (int rc = enqueue_step(b, cfl, with_sources, parity)) return rc;
      continue;
    }
    StepGraph& g = b->graphs[parity][b->cur];
    const int cur0 = b->cur;
    if (!g.exec || g.with_sources != with_sources || g.cfl != cfl) {
      if (g.exec) cudaGraphExecDestroy(g.exec);
      g.exec = nullptr;
      cudaGraph_t graph;
      CK(cudaStreamBeginCapture(b->stream, cudaStreamCaptureModeThreadLocal));
      const int rc = enqueue_step(b, cfl, with_sources, parity);
      cudaError_t e = cudaStreamEndCapture(b->stream, &graph);
      if (rc) return rc;
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
      CK(cudaGraphInstantiate(&g.exec, graph, 0));
      cudaGraphDestroy(graph);
      g.with_sources = with_sources;
      g.parity = parity;
      g.cfl = cfl;
      g.cur = b->cur;  // buffer after the step
      b->cur = cur0;
    }
    CK(cudaGraphLaunch(g.exec, b->stream));
    b->cur = g.cur;
  }
  b->dt_valid = true;  // the last step's fused CFL pass computed the next dt
  b->dt_cfl = cfl;
  return 0;
}

int ppmlr_gpu_block_advance(ppmlr_gpu_block* b, double cfl, int with_sources, long step,
                            double* dt_out) {
  if (int rc = run_steps(b, cfl, with_sources, step, 1)) return rc;
  CK(cudaMemcpyAsync(b->h_pinned + 2, b->d_dt_prev, 8, cudaMemcpyDeviceToHost, b->stream));
  if (int rc = check_impl(b, true)) return rc;
  if (dt_out) *dt_out = b->h_pinned[2];
  return 0;
}

int ppmlr_gpu_block_run(ppmlr_gpu_block* b, double cfl, int with_sources, long first_step,
                        long steps, double* time_out) {
  if (steps <= 0) return 0;
  if (time_out) {
    b->h_pinned[3] = *time_out;
    CK(cudaMemcpyAsync(b->d_time, &b->h_pinned[3], 8, cudaMemcpyHostToDevice, b->stream));
  }
  // errors are checked at least every kMaxStepsPerCheck steps: the keys'
  // step field counts from the start of each window and must not wrap
  for (long done = 0; done < steps;) {
    const long k = std::min(steps - done, kMaxStepsPerCheck);
    if (int rc = run_steps(b, cfl, with_sources, first_step + done, k)) return rc;
    if (done + k < steps)
      if (int rc = check_impl(b, true)) return rc;
    done += k;
  }
  CK(cudaMemcpyAsync(b->h_pinned + 7, b->d_time, 8, cudaMemcpyDeviceToHost, b->stream));
  if (int rc = check_impl(b, true)) return rc;
  if (time_out) *time_out = b->h_pinned[7];
  return 0;
}

int ppmlr_gpu_block_pack_face(ppmlr_gpu_block* b, int face, int layers, double* dev_buf) {
  CK(cudaSetDevice(b->device));
  if (face < 0 || face > 5 || layers < 1 || layers > kG) {
    set_error("pack_face: bad face or layer count");
    return PPMLR_INVALID_SPEC;
  }
  const int axis = face / 2;
  const long long work = (long long)layers * b->n[(axis + 1) % 3] * b->n[(axis + 2) % 3];
  pack_kernel<<<grid_for(work), 256, 0, b->stream>>>(planes(cur_buf(b), b->fs), lay_of(b),
                                                       face, layers, dev_buf);
  CK(cudaGetLastError());
  return 0;
}

int ppmlr_gpu_block_unpack_face(ppmlr_gpu_block* b, int face, int layers,
                                const double* dev_buf) {
  b->dt_valid = false;  // state or dt slot changes
  CK(cudaSetDevice(b->device));
  if (face < 0 || face > 5 || layers < 1 || layers > kG) {
    set_error("unpack_face: bad face or layer count");
    return PPMLR_INVALID_SPEC;
  }
  const int axis = face / 2;
  const long long work = (long long)layers * b->n[(axis + 1) % 3] * b->n[(axis + 2) % 3];
  unpack_kernel<<<grid_for(work), 256, 0, b->stream>>>(planes(cur_buf(b), b->fs),
                                                         lay_of(b), face, layers, dev_buf);
  CK(cudaGetLastError());
  return 0;
}

int ppmlr_gpu_block_copy_face(ppmlr_gpu_block* dst, int face, ppmlr_gpu_block* src,
                              int layers) {
  dst->dt_valid = false;  // state or dt slot changes
  CK(cudaSetDevice(dst->device));
  const int axis = face / 2;
  if (dst->n[(axis + 1) % 3] != src->n[(axis + 1) % 3] ||
      dst->n[(axis + 2) % 3] != src->n[(axis + 2) % 3]) {
    set_error("halo slab face span does not match block face");
    return PPMLR_INVALID_SPEC;
  }
  const long long work = (long long)layers * dst->n[(axis + 1) % 3] * dst->n[(axis + 2) % 3];
  copy_face_kernel<<<grid_for(work), 256, 0, dst->stream>>>(
      planes(cur_buf(dst), dst->fs), lay_of(dst), planes(cur_buf(src), src->fs),
      lay_of(src), face, layers);
  CK(cudaGetLastError());
  return 0;
}

int ppmlr_gpu_block_begin(ppmlr_gpu_block* b, double cfl, long first_step) {
  b->dt_valid = false;  // state or dt slot changes
  if (int rc = deferred(b)) return rc;
  CK(cudaSetDevice(b->device));
  unsigned long long init[2] = {kNoError, 0};
  CK(cudaMemcpyAsync(b->d_err, init, sizeof init, cudaMemcpyHostToDevice, b->stream));
  b->step_base = first_step;
  if (int rc = launch_cfl(b, 0)) return rc;
  return launch_step_end(b, cfl, 0, 1);
}

int ppmlr_gpu_block_sweep_async(ppmlr_gpu_block* b, int axis, int order_index) {
  return ppmlr_gpu_block_sweep_part(b, axis, order_index, 0);
}

int ppmlr_gpu_block_sweep_part(ppmlr_gpu_block* b, int axis, int order_index, int part) {
  b->dt_valid = false;  // state or dt slot changes
  CK(cudaSetDevice(b->device));
  if (axis < 0 || axis > 2 || order_index < 0 || order_index > 2 || part < 0 || part > 2) {
    set_error("sweep_async: bad axis/order/part");
    return PPMLR_INVALID_SPEC;
  }
  return timed_sweep(b, axis, kPhaseSweep0 + order_index, part);
}

int ppmlr_gpu_block_end_step(ppmlr_gpu_block* b, double cfl, int with_sources) {
  return ppmlr_gpu_block_end_step_part(b, cfl, with_sources, 0);
}

int ppmlr_gpu_block_end_step_part(ppmlr_gpu_block* b, double cfl, int with_sources, int part) {
  b->dt_valid = false;  // state or dt slot changes
  CK(cudaSetDevice(b->device));
  if (part < 0 || part > 2) {
    set_error("end_step: bad part");
    return PPMLR_INVALID_SPEC;
  }
  if (with_sources) {
    if (int rc = launch_sources(b, 1, part)) return rc;
    if (part == 1) return 0;  // the interior part closes the step
  } else {
    if (part == 1) return 0;
    if (int rc = launch_frozen(b)) return rc;
    if (int rc = launch_cfl(b, 1)) return rc;
  }
  return launch_step_end(b, cfl, 1, 1);
}

int ppmlr_gpu_block_time(ppmlr_gpu_block* b, double* time_out) {
  CK(cudaSetDevice(b->device));
  CK(cudaMemcpyAsync(b->h_pinned + 5, b->d_time, 8, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  *time_out = b->h_pinned[5];
  return 0;
}

void* ppmlr_gpu_block_stream(ppmlr_gpu_block* b) { return b->stream; }

int ppmlr_gpu_block_set_stream(ppmlr_gpu_block* b, void* stream) {
  CK(cudaSetDevice(b->device));
  CK(cudaStreamSynchronize(b->stream));
  if (b->own_stream) cudaStreamDestroy(b->stream);
  b->stream = static_cast<cudaStream_t>(stream);
  b->own_stream = false;
  drop_step_graphs(b);
  return 0;
}

int ppmlr_gpu_block_synchronize(ppmlr_gpu_block* b) {
  CK(cudaSetDevice(b->device));
  CK(cudaStreamSynchronize(b->stream));
  return 0;
}

int ppmlr_gpu_block_state_view(ppmlr_gpu_block* b, double** field_planes, long long* strides,
                               int* dims) {
  for (int f = 0; f < 8; ++f) field_planes[f] = cur_buf(b) + (long long)f * b->fs;
  strides[0] = 1;
  strides[1] = b->sy;
  strides[2] = b->sz;
  for (int a = 0; a < 3; ++a) dims[a] = b->S[a];
  return kG;
}

int ppmlr_gpu_block_init_ic(ppmlr_gpu_block* b, int kind, const double* params) {
  if (!device_init_supported(kind) || kind < 0) {
    set_error("block_init_ic: kind must be 0..3 (device-evaluated ICs)");
    return PPMLR_INVALID_SPEC;
  }
  if (int rc = block_set_frozen(b, nullptr, nullptr, 0)) return rc;
  double p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (params) std::memcpy(p, params, sizeof p);
  return block_init_device(b, kind, p, true);
}

int ppmlr_gpu_block_dipole_view(ppmlr_gpu_block* b, double** bd_planes) {
  for (int a = 0; a < 3; ++a) bd_planes[a] = b->bd ? b->bd + (long long)a * b->fs : nullptr;
  return b->bd ? 1 : 0;
}

int ppmlr_gpu_block_timing(ppmlr_gpu_block* b, int enable, double* sweep_ms, double* total_ms,
                           long* launches) {
  CK(cudaSetDevice(b->device));
  auto& t = b->timing;
  CK(cudaStreamSynchronize(b->stream));
  double sum = 0.0;
  for (size_t i = 0; i + 1 < t.used; i += 2) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, t.pool[i], t.pool[i + 1]));
    sum += ms;
  }
  if (sweep_ms) *sweep_ms = sum;
  if (launches) *launches = (long)(t.used / 2);
  if (total_ms) *total_ms = (double)b->kernel_launches;  // kernel launch count since reset
  t.used = 0;
  b->kernel_launches = 0;
  t.enabled = enable != 0;
  return 0;
}

}  // extern "C"

namespace {
// strip_max_dt (ppm1d.cpp:307-315) over a batch of strips: min over every
// interior cell of dx / (|v_dir| + c_f,dir), physics::fast_speed in xyz
// order with the plain IEEE operations (ExactOps); NaN candidates drop out
// like std::min's, and the min of the per-strip minima is the global one.
template <int DIR>
__global__ void strip_dt_kernel(const double* __restrict__ st, const double* __restrict__ bd,
                                const double* __restrict__ dx, int n, int g, int ns, Consts cc,
                                unsigned long long* out) {
  const KC k = make_kc(cc);
  const long long total = (long long)ns * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long strip = t / n;
    const int i = (int)(t - strip * n);
    const long long idx = strip * (n + 2 * g) + g + i;
    const double* s = st + 8 * idx;
    const double b0 = bd ? bd[3 * idx] : 0.0, b1 = bd ? bd[3 * idx + 1] : 0.0,
                 b2 = bd ? bd[3 * idx + 2] : 0.0;
    ExactOps o;
    const double cf = fast_speed3<DIR>(s, b0, b1, b2, k, o);
    const double speed = fabs(s[1 + DIR]) + cf;
    const double cand = dx[g + i] / speed;
    if (cand < INFINITY) atomicMin(out, (unsigned long long)__double_as_longlong(cand));
  }
}
}  // namespace

extern "C" {

int ppmlr_gpu_strip_max_dt(const double* states, const double* bd, const double* dx, int n,
                           int ghost, int nstrips, int dir, double gamma, double mu0,
                           int device, double* dt_out) {
  if (n < 1 || ghost < 0 || nstrips < 1 || dir < 0 || dir > 2) {
    set_error("strip_max_dt: bad strip description");
    return PPMLR_INVALID_SPEC;
  }
  CK(cudaSetDevice(device));
  const size_t nn = (size_t)n + 2 * ghost, cells = nn * nstrips;
  double *d_st = nullptr, *d_bd = nullptr, *d_dx = nullptr;
  unsigned long long* d_out = nullptr;
  auto release = [&] {
    cudaFree(d_st);
    cudaFree(d_bd);
    cudaFree(d_dx);
    cudaFree(d_out);
  };
  cudaError_t e = cudaMalloc(&d_st, cells * 64);
  if (e == cudaSuccess && bd) e = cudaMalloc(&d_bd, cells * 24);
  if (e == cudaSuccess) e = cudaMalloc(&d_dx, nn * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_out, 8);
  if (e == cudaSuccess) e = cudaMemcpy(d_st, states, cells * 64, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && bd) e = cudaMemcpy(d_bd, bd, cells * 24, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_dx, dx, nn * 8, cudaMemcpyHostToDevice);
  const unsigned long long inf = kInfBits;
  if (e == cudaSuccess) e = cudaMemcpy(d_out, &inf, 8, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    release();
    return cuda_fail(e, "strip_max_dt setup");
  }
  Consts c{};
  c.gamma = gamma;
  c.mu0 = mu0;
  c.gm1 = gamma - 1.0;
  c.two_mu0 = 2.0 * mu0;
  const long long work = (long long)n * nstrips;
  switch (dir) {
    case 0: strip_dt_kernel<0><<<grid_for(work), 256>>>(d_st, d_bd, d_dx, n, ghost, nstrips, c, d_out); break;
    case 1: strip_dt_kernel<1><<<grid_for(work), 256>>>(d_st, d_bd, d_dx, n, ghost, nstrips, c, d_out); break;
    default: strip_dt_kernel<2><<<grid_for(work), 256>>>(d_st, d_bd, d_dx, n, ghost, nstrips, c, d_out); break;
  }
  unsigned long long bits = inf;
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(&bits, d_out, 8, cudaMemcpyDeviceToHost);
  release();
  if (e != cudaSuccess) return cuda_fail(e, "strip_max_dt");
  std::memcpy(dt_out, &bits, 8);
  return 0;
}

int ppmlr_gpu_sweep_strips(double* states, const double* bd, const double* dx, int n,
                           int ghost, int nstrips, int dir, double dt, double gamma,
                           double mu0, double pressure_floor, int precision, int device) {
  if (n < 1 || nstrips < 1 || ghost < 4 || dir < 0 || dir > 2) {
    set_error("sweep_strips: bad arguments");
    return PPMLR_INVALID_SPEC;
  }
  // A block whose `dir` axis is the strip and whose (dir+1) axis enumerates
  // the strips; ghost cells are the caller's (no boundary fill).
  const int nn = n + 2 * ghost;
  std::vector<double> zero_c(std::max(nstrips, 1) + 2 * ghost, 0.0),
      one_s(std::max(nstrips, 1) + 2 * ghost, 1.0), cen(nn);
  for (int i = 0; i < nn; ++i) cen[i] = i;
  ppmlr_gpu_block_desc d{};
  const int t1 = (dir + 1) % 3, t2 = (dir + 2) % 3;
  d.n[dir] = n;
  d.n[t1] = nstrips;
  d.n[t2] = 1;
  d.ghost = ghost;
  std::vector<double> c1(nstrips + 2 * ghost), s1(nstrips + 2 * ghost, 1.0), c2(1 + 2 * ghost),
      s2(1 + 2 * ghost, 1.0);
  d.centers[dir] = cen.data();
  d.spacings[dir] = dx;
  d.centers[t1] = c1.data();
  d.spacings[t1] = s1.data();
  d.centers[t2] = c2.data();
  d.spacings[t2] = s2.data();
  d.gamma = gamma;
  d.mu0 = mu0;
  d.pressure_floor = pressure_floor;
  d.with_dipole = bd != nullptr;
  d.precision = precision;
  d.device = device;
  ppmlr_gpu_block* b = nullptr;
  if (int rc = ppmlr_gpu_block_create(&d, &b)) return rc;
  // Scatter strips into a ghost-inclusive reference-layout array.
  const int S0 = d.n[0] + 2 * ghost, S1 = d.n[1] + 2 * ghost, S2 = d.n[2] + 2 * ghost;
  std::vector<double> f((size_t)S0 * S1 * S2 * 8, 1.0), bdv;
  if (bd) bdv.assign((size_t)S0 * S1 * S2 * 3, 0.0);
  auto lin = [&](int q, int s) {
    int c[3];
    c[dir] = q;            // 0..nn-1 (ghost-inclusive)
    c[t1] = s + ghost;
    c[t2] = ghost;
    return (size_t)c[0] + (size_t)S0 * (c[1] + (size_t)S1 * c[2]);
  };
  for (int s = 0; s < nstrips; ++s)
    for (int q = 0; q < nn; ++q) {
      const size_t l = lin(q, s);
      std::memcpy(&f[8 * l], states + ((size_t)s * nn + q) * 8, 64);
      if (bd) std::memcpy(&bdv[3 * l], bd + ((size_t)s * nn + q) * 3, 24);
    }
  int rc = ppmlr_gpu_block_upload(b, f.data(), bd ? bdv.data() : nullptr, nullptr, nullptr, 0);
  if (!rc) {
    b->step_base = 0;
    rc = ppmlr_gpu_block_sweep(b, dir, dt);
  }
  if (!rc) {
    // error keys of a bare sweep: phase Sweep0 + dir maps back to `dir`
    unsigned long long key = 0;
    cudaStreamSynchronize(b->stream);
    cudaMemcpy(&key, b->d_err, 8, cudaMemcpyDeviceToHost);
    if (key != kNoError) {
      std::string msg;
      rc = decode_error(b, key, msg);
      // strip-level message: drop the " in sweep axis" suffix and report the
      // sweep_1d exception kind (StepRejected vs UnphysicalState)
      const size_t cut = msg.find(" in sweep axis");
      const std::string inner = cut == std::string::npos ? msg : msg.substr(0, cut);
      set_error(inner);
      rc = inner.rfind("Lagrangian interfaces crossed", 0) == 0 ? PPMLR_STEP_REJECTED
                                                                  : PPMLR_UNPHYSICAL;
      // report the first failing strip (pencil order = strip index)
    }
  }
  if (!rc) rc = ppmlr_gpu_block_download(b, f.data());
  if (!rc)
    for (int s = 0; s < nstrips; ++s)
      for (int q = ghost; q < ghost + n; ++q)
        std::memcpy(states + ((size_t)s * nn + q) * 8, &f[8 * lin(q, s)], 64);
  ppmlr_gpu_block_destroy(b);
  return rc;
}

}  // extern "C"

// ------------------------------------------------------------------
// FP64 pipe peak: independent DFMA chains (MEASURED_PEAKS.json carries no
// FP64 figure; SURVEY.md §8(d) asks for a measured denominator).
namespace {
__global__ void dfma_peak_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}
}  // namespace

extern "C" int ppmlr_gpu_fp64_peak(int device, double* tflops) {
  CK(cudaSetDevice(device));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  double* d = nullptr;
  CK(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000, threads = 512, blocks = sms * 4;
  dfma_peak_kernel<<<blocks, threads>>>(d, 1000, 0.999999, 1e-7);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    dfma_peak_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (err != cudaSuccess) return cuda_fail(err, "dfma_peak_kernel");
  const double flops = 2.0 * 8.0 * (double)iters * threads * blocks;
  *tflops = flops / (best * 1e-3) / 1e12;
  return 0;
}

// ------------------------------------------------------------------
// Self-test of the shared-reciprocal division against the compiler's `/`
// (bit patterns; NaN == NaN).  Operands mix random bit patterns, values of
// physical magnitude, signed zeros, denormals and extremes.
namespace {
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}
__device__ double pick(unsigned long long h, unsigned long long h2) {
  switch (h2 % 8) {
    case 0: return __longlong_as_double((long long)h);                       // any bits
    case 1: return (double)((long long)(h >> 11)) * 1e-12 - 4.6e6;           // physical
    case 2: return ldexp((double)(h >> 11) * 0x1p-53, (int)(h2 >> 8) % 200 - 100);
    case 3: return (h & 1) ? 0.0 : -0.0;
    case 4: return __longlong_as_double((long long)(h & 0x800fffffffffffffull));  // denormal
    case 5: return ldexp(1.0 + (double)(h >> 12) * 0x1p-52, 1000 + (int)(h2 >> 8) % 24);
    case 6: return ldexp(1.0 + (double)(h >> 12) * 0x1p-52, -1000 - (int)(h2 >> 8) % 74);
    default: return (double)(long long)(h % 2001) - 1000.0;                  // small ints
  }
}
__global__ void div_selftest_kernel(long long n, unsigned long long seed,
                                    unsigned long long* bad, double* example) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long h = mix64(seed + 2 * (unsigned long long)i);
    const unsigned long long g = mix64(seed + 2 * (unsigned long long)i + 1);
    const double a = pick(h, mix64(h));
    const double b = pick(g, mix64(g ^ 0x9e3779b97f4a7c15ull));
    const double want = a / b;
    const double got = div_r(a, b, rcp_refined(b));
    const bool same = (__double_as_longlong(want) == __double_as_longlong(got)) ||
                      (isnan(want) && isnan(got));
    if (!same) {
      if (atomicAdd(bad, 1ull) == 0) {
        example[0] = a;
        example[1] = b;
        example[2] = want;
        example[3] = got;
      }
    }
  }
}
}  // namespace

extern "C" int ppmlr_gpu_selftest_division(int device, long long n, unsigned long long seed,
                                           long long* mismatches, double* example4) {
  CK(cudaSetDevice(device));
  unsigned long long* d = nullptr;
  CK(cudaMalloc(&d, 8 + 4 * 8));
  CK(cudaMemset(d, 0, 40));
  div_selftest_kernel<<<148 * 16, 256>>>(n, seed, d, reinterpret_cast<double*>(d + 1));
  CK(cudaGetLastError());
  unsigned long long host[5];
  CK(cudaMemcpy(host, d, 40, cudaMemcpyDeviceToHost));
  cudaFree(d);
  *mismatches = (long long)host[0];
  if (example4) std::memcpy(example4, host + 1, 32);
  return 0;
}
