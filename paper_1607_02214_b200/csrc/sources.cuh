// apply_sources + restore_frozen_core + the next step's compute_dt
// (proj/src/stepper.cpp:119-200, 284-286) as stencil kernels, compiled once
// per precision mode (PPMLR_KNS = strict | fast; see exact_div.cuh).
#pragma once
#include <cuda.h>  // CUtensorMap

#include "grid_types.cuh"
#include "ppmlr_dev.cuh"

namespace ppmlr_b200 {

// TMA descriptors of the source kernel's plane loads: v, B' (and the
// dipole) of the source buffer, 3-D tensors over the padded block with the
// box of one z plane of a tile plus its x/y halo ({34, 10, 1}).
struct SrcMaps {
  CUtensorMap f[9];
};

struct SrcArgs {
  Planes in, out;
  Lay L;
  const double *bd0, *bd1, *bd2;
  const double *hm0, *hp0, *hm1, *hp1, *hm2, *hp2;  // per axis, ghost-inclusive
  const double *den0, *den1, *den2, *rden0, *rden1, *rden2;
  const double *dx0, *dx1, *dx2;
  // frozen core
  int fl0, fl1, fl2, fn0, fn1, fn2;
  const int* fslot;
  const double* fst;
  long long nfrozen;
  Consts c;
  CtxPtrs ctx;
  int fuse_cfl;
  unsigned* redo_count;
  unsigned* redo_list;
  unsigned redo_cap;
  int part, cl, cr;  // x-tile split of a part launch (sweep.cuh split_*)
};

namespace PPMLR_KNS {

// the (x, y) tile of sources_tiled_kernel and its halo box (see below)
constexpr int kSrcTX = 32, kSrcTY = 8, kSrcHX = kSrcTX + 4, kSrcHY = kSrcTY + 2;

#ifdef PPMLR_FAST_MATH
using SrcOps = FastMathOps;
#else
using SrcOps = FastOps;
#endif

// The three CFL candidates of compute_dt (stepper.cpp:128-137) for one cell.
// Returns false (and the failing axis) on a non-finite candidate.
template <class Ops>
__device__ __forceinline__ void cfl_cands(const double* s, double b0, double b1, double b2,
                                          double d0, double d1, double d2, const KC& c, Ops& o,
                                          double* cand) {
  double cf[3];
  fast_speed3_all(s, b0, b1, b2, c, o, cf);
  cand[0] = o.dv(d0, fabs(s[1]) + cf[0]);
  cand[1] = o.dv(d1, fabs(s[2]) + cf[1]);
  cand[2] = o.dv(d2, fabs(s[3]) + cf[2]);
}

__device__ __forceinline__ bool cfl_cell(const double* s, double b0, double b1, double b2,
                                         double d0, double d1, double d2, const KC& c,
                                         double& mn, int& bad_axis) {
  double cand[3];
  SrcOps fo;
  cfl_cands(s, b0, b1, b2, d0, d1, d2, c, fo, cand);
  if (fo.bad) {
    ExactOps eo;
    cfl_cands(s, b0, b1, b2, d0, d1, d2, c, eo, cand);
  }
  for (int a = 0; a < 3; ++a)
    if (!isfinite(cand[a])) {
      bad_axis = a;
      return false;
    }
  mn = smin(smin(smin(mn, cand[0]), cand[1]), cand[2]);
  return true;
}

// stepper.cpp:42-45; den = (hm*hp)*(hm+hp) and its refined reciprocal come
// from per-position geometry tables.
template <class Ops>
__device__ __forceinline__ double central_diff(double fm, double f0, double fp, double hm,
                                               double hp, double den, double rden, Ops& o) {
  return o.div(((hm * hm) * fp + ((hp * hp) - (hm * hm)) * f0) - (hp * hp) * fm, den, rden);
}

// apply_sources (stepper.cpp:141-200) for one cell from its 7-point
// stencil: own state s[8] and dipole bo[3]; per axis a the minus/plus
// neighbours' v and B' (nv[a][side][0..5]) and dipole (nbd[a][side][0..2]);
// the axis geometry hm, hp, den = (hm*hp)*(hm+hp), rden.  Writes the
// updated primitive state to q; returns cons_to_prim's code.
template <class Ops>
__device__ __forceinline__ int source_update(const double* s, const double* bo,
                                             const double (*nv)[2][6],
                                             const double (*nbd)[2][3], const double* hm,
                                             const double* hp, const double* den,
                                             const double* rden, const KC& c, double dt,
                                             Ops& o, double* q) {
  double gb[3][3], ge[3][3];
  double e0[3];
  cross3(s[1], s[2], s[3], bo[0], bo[1], bo[2], e0);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double em[3], ep[3];
    cross3(nv[a][0][0], nv[a][0][1], nv[a][0][2], nbd[a][0][0], nbd[a][0][1], nbd[a][0][2], em);
    cross3(nv[a][1][0], nv[a][1][1], nv[a][1][2], nbd[a][1][0], nbd[a][1][1], nbd[a][1][2], ep);
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) {
      gb[a][comp] = central_diff(nv[a][0][3 + comp], s[4 + comp], nv[a][1][3 + comp], hm[a], hp[a],
                                 den[a], rden[a], o);
      ge[a][comp] = central_diff(em[comp], e0[comp], ep[comp], hm[a], hp[a], den[a], rden[a], o);
    }
  }
  const double cb0 = gb[1][2] - gb[2][1], cb1 = gb[2][0] - gb[0][2], cb2 = gb[0][1] - gb[1][0];
  const double ce0 = ge[1][2] - ge[2][1], ce1 = ge[2][0] - ge[0][2], ce2 = ge[0][1] - ge[1][0];
  const double div_b = (gb[0][0] + gb[1][1]) + gb[2][2];
  double sm[3];
  cross3(cb0, cb1, cb2, bo[0], bo[1], bo[2], sm);
  sm[0] = o.div(sm[0], c.c.mu0, c.r_mu0);
  sm[1] = o.div(sm[1], c.c.mu0, c.r_mu0);
  sm[2] = o.div(sm[2], c.c.mu0, c.r_mu0);
  const double si0 = ce0 - s[1] * div_b, si1 = ce1 - s[2] * div_b, si2 = ce2 - s[3] * div_b;
  const double se = ((s[1] * sm[0] + s[2] * sm[1]) + s[3] * sm[2]) +
                    o.div((s[4] * ce0 + s[5] * ce1) + s[6] * ce2, c.c.mu0, c.r_mu0);
  double u[8];
  prim_to_cons3(s, u, c, o);
  u[1] = u[1] + sm[0] * dt;
  u[2] = u[2] + sm[1] * dt;
  u[3] = u[3] + sm[2] * dt;
  u[4] = u[4] + si0 * dt;
  u[5] = u[5] + si1 * dt;
  u[6] = u[6] + si2 * dt;
  u[7] = u[7] + dt * se;
  return cons_to_prim3(u, q, c, o);
}



// Gathers one cell's 7-point stencil from global memory (EXACT re-run and
// reference path of the tiled kernel below).
template <bool DIPOLE>
__device__ __forceinline__ void gather_stencil(const SrcArgs& A, int i, int j, int k, double* s,
                                               double* bo, double (*nv)[2][6],
                                               double (*nbd)[2][3], double* hm, double* hp,
                                               double* den, double* rden) {
  const Lay& L = A.L;
  const long long d = L.idx(i, j, k);
#pragma unroll
  for (int f = 0; f < 8; ++f) s[f] = A.in.f[f][d];
  bo[0] = DIPOLE ? A.bd0[d] : 0.0;
  bo[1] = DIPOLE ? A.bd1[d] : 0.0;
  bo[2] = DIPOLE ? A.bd2[d] : 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const long long st = a == 0 ? 1 : (a == 1 ? L.sy : L.sz);
    const int lc = (a == 0 ? i : (a == 1 ? j : k)) + kG;
    hm[a] = (a == 0 ? A.hm0 : (a == 1 ? A.hm1 : A.hm2))[lc];
    hp[a] = (a == 0 ? A.hp0 : (a == 1 ? A.hp1 : A.hp2))[lc];
    den[a] = (a == 0 ? A.den0 : (a == 1 ? A.den1 : A.den2))[lc];
    rden[a] = (a == 0 ? A.rden0 : (a == 1 ? A.rden1 : A.rden2))[lc];
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const long long dn = side == 0 ? d - st : d + st;
#pragma unroll
      for (int f = 0; f < 6; ++f) nv[a][side][f] = A.in.f[1 + f][dn];
      nbd[a][side][0] = DIPOLE ? A.bd0[dn] : 0.0;
      nbd[a][side][1] = DIPOLE ? A.bd1[dn] : 0.0;
      nbd[a][side][2] = DIPOLE ? A.bd2[dn] : 0.0;
    }
  }
}

// Epilogue shared by both source kernels: error key, frozen-core override
// (restore_frozen_core), store, and the next step's CFL candidates.
template <bool DIPOLE>
__device__ __forceinline__ void source_epilogue(const SrcArgs& A, const KC& c, int i, int j,
                                                int k, long long t, const double* s,
                                                const double* bo, double* q, int bad,
                                                unsigned long long step, double& mn,
                                                double d0, double d1, double d2) {
  const Lay& L = A.L;
  if (bad) {
    atomicMin(A.ctx.err, err_key(step, kPhaseSources, 0,
                                 ((unsigned long long)t << 2) |
                                     (bad == 1 ? kErrDensity : kErrPressure)));
#pragma unroll
    for (int f = 0; f < 8; ++f) q[f] = s[f];
  }
  if (A.nfrozen > 0) {
    const int fi = i - A.fl0, fj = j - A.fl1, fk = k - A.fl2;
    if (fi >= 0 && fi < A.fn0 && fj >= 0 && fj < A.fn1 && fk >= 0 && fk < A.fn2) {
      const int slot = A.fslot[fi + A.fn0 * (fj + A.fn1 * fk)];
      if (slot >= 0) {
#pragma unroll
        for (int f = 0; f < 8; ++f) q[f] = A.fst[f * A.nfrozen + slot];
      }
    }
  }
  const long long d = L.idx(i, j, k);
#pragma unroll
  for (int f = 0; f < 8; ++f) A.out.f[f][d] = q[f];
  if (A.fuse_cfl) {
    int badax = 0;
    if (!cfl_cell(q, bo[0], bo[1], bo[2], d0, d1, d2, c, mn, badax))
      atomicMin(A.ctx.err, err_key(step + 1, kPhaseCfl, 0, ((unsigned long long)t * 3 + badax) << 2));
  }
}

// EXACT re-run of the cells queued by the tiled kernel (redo list; on
// overflow every cell), with plain `/` and `sqrt`.
template <bool DIPOLE>
__global__ void __launch_bounds__(256, 2) sources_exact_kernel(const SrcArgs A) {
  const Lay& L = A.L;
  const KC c = make_kc(A.c);
  const long long total = (long long)L.n0 * L.n1 * L.n2;
  double mn = __longlong_as_double(kInfBits);
  const unsigned long long step = *A.ctx.step;
  const double dt = *A.ctx.dt;
  const bool all = *A.redo_count > A.redo_cap;
  const long long n_items = all ? total : (long long)*A.redo_count;
  for (long long it = blockIdx.x * (long long)blockDim.x + threadIdx.x; it < n_items;
       it += (long long)gridDim.x * blockDim.x) {
    const long long t = all ? it : (long long)A.redo_list[it];
    const int i = (int)(t % L.n0);
    const int j = (int)((t / L.n0) % L.n1);
    const int k = (int)(t / ((long long)L.n0 * L.n1));
    if (all && A.part) {  // overflow: every cell of this part's x tiles
      const int xt = i / kSrcTX;
      if ((A.part == 1) != (xt < A.cl || xt >= A.cr)) continue;
    }
    double s[8], bo[3], nv[3][2][6], nbd[3][2][3], hm[3], hp[3], den[3], rden[3], q[8];
    gather_stencil<DIPOLE>(A, i, j, k, s, bo, nv, nbd, hm, hp, den, rden);
    ExactOps eo;
    const int bad = source_update(s, bo, nv, nbd, hm, hp, den, rden, c, dt, eo, q);
    source_epilogue<DIPOLE>(A, c, i, j, k, t, s, bo, q, bad, step, mn, A.dx0[i + kG],
                            A.dx1[j + kG], A.dx2[k + kG]);
  }
  if (A.fuse_cfl) block_min_commit(mn, A.ctx.min);
}

// apply_sources (stepper.cpp:141-200) + restore_frozen_core (:284-286) +
// the next step's compute_dt (:119-139), 2.5-D blocked: a CTA owns a 32x8
// (x, y) tile and marches through a z chunk.  The planes of v, B' (and the
// dipole) with a one-cell x/y halo live in a 4-slot shared-memory ring
// filled with cp.async two planes ahead of the plane being updated, so every
// stencil input is fetched from HBM once and its latency is overlapped.
// SrcOps (branch-free fast paths); cells whose guards fail are queued for
// sources_exact_kernel.
// The plane box spans x0-2 .. x0+33: a TMA box must start on a 16-byte
// boundary in x (an even FP64 coordinate), so the x halo is 2 cells wide on
// the left (only x0-1 is read) and 2 on the right.
constexpr int kSrcSlots = 4;
// plane-field stride in the ring, padded to 128 B (the TMA destination rule)
constexpr int kSrcPL = ((kSrcHX * kSrcHY + 15) / 16) * 16;

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// The dipole ring (106 KB) allows 2 CTAs per SM, so registers are not the
// occupancy limit there: bounding them for 3 spilled (strict: 352 B of
// stack).  With 2: C3 / C5 strict +8.6% / +7%, fast C3 +0.8%.
#ifndef PPMLR_SRC_DIPOLE_MINB
#define PPMLR_SRC_DIPOLE_MINB 2
#endif
#ifndef PPMLR_SRC_MINB
#define PPMLR_SRC_MINB 3
#endif
template <bool DIPOLE>
__global__ void __launch_bounds__(kSrcTX * kSrcTY, DIPOLE ? PPMLR_SRC_DIPOLE_MINB : PPMLR_SRC_MINB)
    sources_tiled_kernel(const SrcArgs A, int zchunk, const __grid_constant__ SrcMaps M) {
  constexpr int NF = DIPOLE ? 9 : 6;
  constexpr int PL = kSrcPL;                       // ring stride per plane field
  extern __shared__ __align__(128) double ring[];  // [kSrcSlots][NF][PL]
  __shared__ __align__(8) unsigned long long s_bar[kSrcSlots];
  const Lay& L = A.L;
  const KC c = make_kc(A.c);
  const int tx = threadIdx.x % kSrcTX, ty = threadIdx.x / kSrcTX;
  const int x0 = split_unit(A.part, A.cl, A.cr, blockIdx.x) * kSrcTX, y0 = blockIdx.y * kSrcTY;
  const int z0 = blockIdx.z * zchunk, z1 = min(L.n2, z0 + zchunk);
  const int i = x0 + tx, j = y0 + ty;
  const bool in_xy = i < L.n0 && j < L.n1;
  const unsigned long long step = *A.ctx.step;
  const double dt = *A.ctx.dt;
  double mn = __longlong_as_double(kInfBits);

  // Planes z in [z0-1, z1] exist (the ghost layer at -1 / n2 included).
  // Plane z lives in ring slot r % 4, r = z - (z0 - 1); one elected thread
  // streams it in with TMA (one box per field) completing on that slot's
  // mbarrier, whose phase for plane z is (r / 4) & 1.
  auto slot_of = [&](int z) { return ring + (size_t)((z - z0 + 1) % kSrcSlots) * NF * PL; };
  auto bar_of = [&](int z) {
    return (unsigned)__cvta_generic_to_shared(&s_bar[(z - z0 + 1) % kSrcSlots]);
  };
  auto issue_plane = [&](int z) {  // thread 0 only
    if (z > z1) return;
    const unsigned bar = bar_of(z);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"((unsigned)(NF * kSrcHX * kSrcHY * sizeof(double)))
                 : "memory");
    double* dstp = slot_of(z);
#pragma unroll
    for (int f = 0; f < NF; ++f)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              (unsigned)__cvta_generic_to_shared(dstp + f * PL)),
          "l"(reinterpret_cast<unsigned long long>(&M.f[f])), "r"(x0 - 2 + kG),
          "r"(y0 - 1 + kG), "r"(z + kG), "r"(bar)
          : "memory");
  };
  auto wait_plane = [&](int z) {
    const unsigned bar = bar_of(z), parity = ((z - z0 + 1) / kSrcSlots) & 1;
    unsigned done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
          "selp.b32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(bar), "r"(parity)
          : "memory");
  };
  if (threadIdx.x == 0) {
    for (int q = 0; q < kSrcSlots; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&s_bar[q]))
                   : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    issue_plane(z0 - 1);
    issue_plane(z0);
    issue_plane(z0 + 1);
  }
  __syncthreads();
  wait_plane(z0 - 1);
  wait_plane(z0);
  // per-thread constant geometry along x and y
  double hm[3], hp[3], den[3], rden[3];
  if (in_xy) {
    hm[0] = A.hm0[i + kG];
    hp[0] = A.hp0[i + kG];
    den[0] = A.den0[i + kG];
    rden[0] = A.rden0[i + kG];
    hm[1] = A.hm1[j + kG];
    hp[1] = A.hp1[j + kG];
    den[1] = A.den1[j + kG];
    rden[1] = A.rden1[j + kG];
  }
  const int cc = (ty + 1) * kSrcHX + (tx + 2);  // this cell in a plane
  // per-thread spacings and the z-geometry of the plane, one plane ahead
  const double dxi = in_xy ? A.dx0[i + kG] : 0.0, dxj = in_xy ? A.dx1[j + kG] : 0.0;
  double gn[5] = {A.hm2[z0 + kG], A.hp2[z0 + kG], A.den2[z0 + kG], A.rden2[z0 + kG],
                  A.dx2[z0 + kG]};
  double rho_n = 0.0, p_n = 0.0;                // own rho, p of plane k (prefetched)
  if (in_xy) {
    const long long d = L.idx(i, j, z0);
    rho_n = A.in.f[0][d];
    p_n = A.in.f[7][d];
  }
  for (int k = z0; k < z1; ++k) {
    // the end-of-iteration barrier freed plane k-2's slot for plane k+2
    if (threadIdx.x == 0) issue_plane(k + 2);
    wait_plane(k + 1);
    const double rho_k = rho_n, p_k = p_n;
    double gk[5];
#pragma unroll
    for (int g = 0; g < 5; ++g) gk[g] = gn[g];
    if (k + 1 < z1) {
      gn[0] = A.hm2[k + 1 + kG];
      gn[1] = A.hp2[k + 1 + kG];
      gn[2] = A.den2[k + 1 + kG];
      gn[3] = A.rden2[k + 1 + kG];
      gn[4] = A.dx2[k + 1 + kG];
    }
    if (in_xy && k + 1 < z1) {
      const long long dn = L.idx(i, j, k + 1);
      rho_n = A.in.f[0][dn];
      p_n = A.in.f[7][dn];
    }
    if (in_xy) {
      const double* pm = slot_of(k - 1);
      const double* p0 = slot_of(k);
      const double* pp = slot_of(k + 1);
      double s[8], bo[3], nv[3][2][6], nbd[3][2][3], q[8];
      s[0] = rho_k;
      s[7] = p_k;
#pragma unroll
      for (int f = 0; f < 6; ++f) s[1 + f] = p0[f * PL + cc];
#pragma unroll
      for (int f = 0; f < 3; ++f) bo[f] = DIPOLE ? p0[(6 + f) * PL + cc] : 0.0;
      const int nb_off[2][2] = {{cc - 1, cc + 1}, {cc - kSrcHX, cc + kSrcHX}};
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int side = 0; side < 2; ++side) {
#pragma unroll
          for (int f = 0; f < 6; ++f) nv[a][side][f] = p0[f * PL + nb_off[a][side]];
#pragma unroll
          for (int f = 0; f < 3; ++f)
            nbd[a][side][f] = DIPOLE ? p0[(6 + f) * PL + nb_off[a][side]] : 0.0;
        }
#pragma unroll
      for (int f = 0; f < 6; ++f) {
        nv[2][0][f] = pm[f * PL + cc];
        nv[2][1][f] = pp[f * PL + cc];
      }
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        nbd[2][0][f] = DIPOLE ? pm[(6 + f) * PL + cc] : 0.0;
        nbd[2][1][f] = DIPOLE ? pp[(6 + f) * PL + cc] : 0.0;
      }
      hm[2] = gk[0];
      hp[2] = gk[1];
      den[2] = gk[2];
      rden[2] = gk[3];
      SrcOps fo;
      const int bad = source_update(s, bo, nv, nbd, hm, hp, den, rden, c, dt, fo, q);
      const long long t = (long long)i + (long long)L.n0 * ((long long)j + (long long)L.n1 * k);
      if (fo.bad) {
        const unsigned slot = atomicAdd(A.redo_count, 1u);
        if (slot < A.redo_cap) A.redo_list[slot] = (unsigned)t;
      } else {
        source_epilogue<DIPOLE>(A, c, i, j, k, t, s, bo, q, bad, step, mn, dxi, dxj, gk[4]);
      }
    }
    __syncthreads();  // plane k-1's slot is refilled next iteration
  }
  if (A.fuse_cfl) block_min_commit(mn, A.ctx.min);
}

}  // namespace PPMLR_KNS
}  // namespace ppmlr_b200
