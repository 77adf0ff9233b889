// Persistent, prefetching schedule of the directional PPMLR sweep (both
// builds, compile-time tile, with or without the dipole): the same per-pencil algorithm as sweep.cuh's
// sweep_tile (proj/src/ppm1d.cpp:111-364, stepper.cpp:249-282) with three
// changes of schedule, measured against the one-shot kernel on the B200:
//
//  * Persistent CTAs (3 per SM) walk the tiles; the tile's 8 input planes
//    arrive by TMA in one of two FLD buffers, and the elected thread issues
//    the NEXT tile's loads when the current tile starts, so the HBM latency
//    of a tile load is hidden behind a whole tile of compute (the one-shot
//    kernel waited for it: ~12% of the sweep's stall samples).
//  * The conserved state is not stored by P0: P7 recomputes it from the
//    zone's own primitives (prim_to_cons, the same expressions), and only
//    tiles with a moving edge write it (into the dead FLD slots) for the
//    remap parabolas.  That frees the 8 slots the prefetch buffer needs:
//    2 x 8 (FLD) + 8 (TR) + 8 (LFT) + 1 (CF) = 33 slots, as before.
//  * The Lagrangian Riemann problem at edge s+1 is solved by the thread of
//    zone s, which still holds that zone's traced RIGHT state in registers:
//    the right states never go through shared memory and the write-after-
//    read barrier in the middle of P3 disappears.
//
// Phases and barriers of one tile (non-moving tiles skip P7b/P8):
//   [TMA wait] P0 | P3 | P4 (+moving vote) | P7 | P7b | P8 | slivers | P9 | close
//   P0   strip-frame prim -> cf (CF), primitive slopes (TR)
//   P3   traced states: left -> LFT, right kept in registers
//   P4   edge s+1: u* -> CF[s+1], flux -> TR[s+1]
//   P7   Lagrangian update -> lag (LFT); moving tiles: cons -> FLD
//   P7b  moving: conserved slopes -> TR
//   P8   moving: slivers (registers), then -> TR
//   P9   remap + cons_to_prim -> FLD (TMA box store) or global
#pragma once
#include "sweep.cuh"

namespace ppmlr_b200 {
namespace PPMLR_KNS {

#ifndef PPMLR_SWEEP_V2_RSMEM
// The traced right states go through the idle FLD buffer (the next tile's
// fields are requested after P4 instead of at the tile start: the load still
// has most of the tile to land) instead of being held in registers across
// P3's barrier.
#ifdef PPMLR_FAST_MATH
#define PPMLR_SWEEP_V2_RSMEM 1  // measured: fast blast -0.4%, C5 -1.2%, C2 -1.6% sweep time
#else
#define PPMLR_SWEEP_V2_RSMEM 0  // strict: +2.9% on the blast (kept in registers)
#endif
#endif

// z sweeps: right states in registers and the next tile's fields requested
// at the tile start.  A z result box (64 rows of 32 B, 64 planes apart)
// takes long to drain through the TMA store; with the right states in the
// other buffer every warp waited for it before P3 (the largest stall of
// the blast z sweep, profiles/r02).  Blast sweep -0.8%, C5 neutral; a
// request after P4 instead: -0.1%.
#ifndef PPMLR_SWEEP_V2_RSMEM_AXES
#define PPMLR_SWEEP_V2_RSMEM_AXES 3  // bit a: axis a keeps right states in shared memory
#endif
#ifndef PPMLR_SWEEP_V2_LATE_PF_Z
#define PPMLR_SWEEP_V2_LATE_PF_Z 0
#endif
template <int AXIS>
__device__ constexpr bool rs_of() {
  return PPMLR_SWEEP_V2_RSMEM && ((PPMLR_SWEEP_V2_RSMEM_AXES >> AXIS) & 1);
}
template <int AXIS>
__device__ constexpr bool late_pf() {
  return rs_of<AXIS>() || (AXIS == 2 && PPMLR_SWEEP_V2_LATE_PF_Z);
}

#ifndef PPMLR_SWEEP_X_BD_EARLY
#define PPMLR_SWEEP_X_BD_EARLY 1  // x sweeps with the dipole: C5 / C3 fast +0.3%
#endif
#ifndef PPMLR_SWEEP_BD_BRICKS
#define PPMLR_SWEEP_BD_BRICKS 1  // z sweeps read B_d from its z-brick copy (SweepArgs::bdz)
#endif
#ifndef PPMLR_SWEEP_BD_BRICKS_Y
#define PPMLR_SWEEP_BD_BRICKS_Y 1  // ... and y sweeps from a y-brick copy
#endif

template <int AXIS, bool DIPOLE, int NP, int TL, class Ops, class Prefetch, class Sync>
__device__ __forceinline__ bool sweep_tile_v2(const SweepArgs& A, const SweepMaps& M,
                                              const TileId id, double* smem, double* FLD,
                                              double* RSB, unsigned long long* s_err,
                                              bool& stored, const Prefetch& prefetch,
                                              const Sync& lsync, bool& moved) {
  bool tbad = false;
  // TL > 0: the compile-time tile; TL == 0: the block's runtime tile L + 8
  const int TLr = TL > 0 ? TL : A.L + 8;
  const int NT = NP * TLr;
  const int T = slot_stride(NT);
  double* TR = smem + 16 * T;
  double* LFT = smem + 24 * T;
  double* CF = smem + 32 * T;
  constexpr int SS = AXIS == 0 ? 1 : NP;
  const int seg = id.seg, grp = id.grp, oc = id.oc;
  const int nn = A.n + 8;
  const int seg0 = seg * A.L;
  const int TLv = min(TLr, nn - seg0);
  const bool final_seg = seg == A.nseg - 1;
  const int zmax = final_seg ? TLv - 2 : TLr - 3;
  const int g0 = grp * NP;
  const int npv = min(NP, A.ng - g0);
  const bool whole = TLv == TLr && npv == NP;
  const double dt = *A.dt;
  const Consts& c = A.c;
  const KC k = make_kc(c);
  const int ci = threadIdx.x;
  int s, p;
  if (AXIS == 0) {
    p = ci / TLr;
    s = ci - p * TLr;
  } else {
    s = ci / NP;
    p = ci - s * NP;
  }
  const bool live = ci < NT && p < npv;
  const int q = seg0 + s;
  auto pencil_index = [&]() -> unsigned long long {
    const int gcoord = g0 + p;
    const int t1 = AXIS == 1 ? oc : gcoord;
    const int t2 = AXIS == 1 ? gcoord : oc;
    return (unsigned long long)t1 + (unsigned long long)A.nb * (unsigned long long)t2;
  };
  constexpr int a = AXIS, b = (AXIS + 1) % 3, d = (AXIS + 2) % 3;
  constexpr bool kBricks =
      (AXIS == 2 && PPMLR_SWEEP_BD_BRICKS) || (AXIS == 1 && PPMLR_SWEEP_BD_BRICKS_Y);
  constexpr int fof[8] = {0, 1 + a, 1 + b, 1 + d, 4 + a, 4 + b, 4 + d, 7};

  // ---- P0: cf and primitive slopes ----------------------------------------
  if (DIPOLE && AXIS == 0 && PPMLR_SWEEP_X_BD_EARLY && live && s < TLv) {
    // x sweeps: B_d loads issued first, in flight during the slopes
    const long long off = (long long)(g0 + p + 4) * A.stride_g +
                          (long long)(oc + 4) * A.stride_o + (long long)q * A.stride_a;
    const double b0 = __ldg(A.bd[0] + off), b1 = __ldg(A.bd[1] + off),
                 b2 = __ldg(A.bd[2] + off);
    if (s >= 1 && s <= TLv - 2) {
      const SlopeC sc = slope_coef(A.slope, q);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const double* pv = FLD + fof[v] * T + ci;
        TR[v * T + ci] = slope_with(pv[-SS], pv[0], pv[SS], sc);
      }
    }
    double qv[8];
#pragma unroll
    for (int f = 0; f < 8; ++f) qv[f] = FLD[f * T + ci];
    Ops o;
    CF[ci] = fast_speed3<AXIS, Ops, true>(qv, b0, b1, b2, k, o);
    tbad |= o.bad;
  } else if (live && s < TLv) {
    double qv[8];
#pragma unroll
    for (int f = 0; f < 8; ++f) qv[f] = FLD[f * T + ci];
    Ops o;
    if (DIPOLE && kBricks) {  // B_d bricks along the sweep axis (coalesced)
      const long long zo = ((long long)(oc * A.bdz_ngx + grp) * A.bdz_s2 + q) * 4 + p;
      CF[ci] = fast_speed3<AXIS, Ops, true>(qv, __ldg(A.bdz + zo), __ldg(A.bdz + A.bdz_cs + zo),
                                            __ldg(A.bdz + 2 * A.bdz_cs + zo), k, o);
    } else if (DIPOLE) {  // B_d from global memory (L1/L2: 3 planes, read twice per sweep)
      const long long off = (long long)(g0 + p + 4) * A.stride_g +
                            (long long)(oc + 4) * A.stride_o + (long long)q * A.stride_a;
      CF[ci] = fast_speed3<AXIS, Ops, true>(qv, __ldg(A.bd[0] + off), __ldg(A.bd[1] + off),
                                            __ldg(A.bd[2] + off), k, o);
    } else {
      CF[ci] = fast_speed3<AXIS, Ops, false>(qv, 0.0, 0.0, 0.0, k, o);
    }
    tbad |= o.bad;
    if (s >= 1 && s <= TLv - 2) {
      const SlopeC sc = slope_coef(A.slope, q);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const double* pv = FLD + fof[v] * T + ci;
        TR[v * T + ci] = slope_with(pv[-SS], pv[0], pv[SS], sc);
      }
    }
  }
  lsync(0);

  // ---- P3: traced states of zones [2, zmax]; L -> LFT, R in registers ------
  double R[8];
  const bool z3 = live && s >= 2 && s <= zmax;
  if (z3) {
    const bool flat = q >= nn - 2;
    double e0[kQfcN], e1[kQfcN];
#pragma unroll
    for (int j = 0; j < kQfcN; ++j) {
      e0[j] = __ldg(A.qfc + kQfcN * q + j);
      e1[j] = __ldg(A.qfc + kQfcN * (q + 1) + j);
    }
    Ops o;
    const double sigma =
        sclamp(o.div(CF[ci] * dt, __ldg(A.dx + q), __ldg(A.rdx + q)), 0.0, 1.0);
    const double hs = 0.5 * sigma;
    const double tw = tw_of(sigma, k, o);
    auto trace = [&](auto F, const int v, double& l, double& r) {
      const double* pv = FLD + fof[v] * T + ci;
      if (!decltype(F)::value) {
        const double* dv = TR + v * T + ci;
        auto win = [&](int j) { return pv[j * SS]; };
        auto dwin = [&](int j) { return dv[j * SS]; };
        zone_traced_dm(win, dwin, e0, e1, k, o, hs, tw, l, r);
      } else if (Ops::kFastMath) {  // flat strip-end zone
        l = pv[0];
        r = pv[0];
      } else {  // the reference's arithmetic on the flat parabola (-0 + 0 = +0)
        l = avg_left(pv[0], pv[0], 0.0, hs, tw);
        r = avg_right(pv[0], pv[0], 0.0, hs, tw);
      }
    };
    auto all8 = [&](auto F) {
      double Lr, Lp;
      trace(F, kRho, Lr, R[kRho]);
      trace(F, kPE, Lp, R[kPE]);
      const bool badL = !(Lr > 0.0) || !(Lp > 0.0);
      const bool badR = !(R[kRho] > 0.0) || !(R[kPE] > 0.0);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        double l = v == kRho ? Lr : Lp;
        if (v != kRho && v != kPE) trace(F, v, l, R[v]);
        LFT[v * T + ci] = l;
      }
      if (badL || badR) {  // rare: the zone falls back to its own state
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const double own = FLD[fof[v] * T + ci];
          if (badL) LFT[v * T + ci] = own;
          if (badR) R[v] = own;
        }
      }
      if (rs_of<AXIS>()) {
#pragma unroll
        for (int v = 0; v < 8; ++v) RSB[v * T + ci] = R[v];
      }
    };
    if (flat)
      all8(FlatTag<true>{});
    else
      all8(FlatTag<false>{});
    tbad |= o.bad;
  }
  lsync(1);

  // ---- P4: edge m = s + 1 in [3, zmax] by the thread of zone s ------------
  bool mv = false;
  if (live && s >= 2 && s <= zmax - 1) {
    double f[8];
    double bl[3] = {0.0, 0.0, 0.0}, br[3] = {0.0, 0.0, 0.0};
    if (DIPOLE && kBricks) {  // bricks, components in strip order (a, b, d)
      const long long zo = ((long long)(oc * A.bdz_ngx + grp) * A.bdz_s2 + q) * 4 + p;
      constexpr int ja = AXIS, jb = (AXIS + 1) % 3, jd = (AXIS + 2) % 3;
      bl[0] = __ldg(A.bdz + ja * A.bdz_cs + zo);
      bl[1] = __ldg(A.bdz + jb * A.bdz_cs + zo);
      bl[2] = __ldg(A.bdz + jd * A.bdz_cs + zo);
      br[0] = __ldg(A.bdz + ja * A.bdz_cs + zo + 4);
      br[1] = __ldg(A.bdz + jb * A.bdz_cs + zo + 4);
      br[2] = __ldg(A.bdz + jd * A.bdz_cs + zo + 4);
    } else if (DIPOLE) {  // the two zones' B_d in strip order (a, b, d)
      const long long off = (long long)(g0 + p + 4) * A.stride_g +
                            (long long)(oc + 4) * A.stride_o + (long long)q * A.stride_a;
      constexpr int ja = AXIS, jb = (AXIS + 1) % 3, jd = (AXIS + 2) % 3;
      bl[0] = __ldg(A.bd[ja] + off);
      bl[1] = __ldg(A.bd[jb] + off);
      bl[2] = __ldg(A.bd[jd] + off);
      br[0] = __ldg(A.bd[ja] + off + A.stride_a);
      br[1] = __ldg(A.bd[jb] + off + A.stride_a);
      br[2] = __ldg(A.bd[jd] + off + A.stride_a);
    }
    const SmemVec qr{LFT + ci + SS, T};
    Ops o;
    double us;
    if (rs_of<AXIS>()) {
      const SmemVec ql{RSB + ci, T};
      us = solve_edge<SmemVec, SmemVec, Ops, DIPOLE>(ql, qr, bl, br, k, f, o);
    } else {
      us = solve_edge<double[8], SmemVec, Ops, DIPOLE>(R, qr, bl, br, k, f, o);
    }
    tbad |= o.bad;
    CF[ci + SS] = us;
    mv = s + 1 >= 4 && s + 1 <= TLv - 4 && us * dt != 0.0;
#pragma unroll
    for (int v = 0; v < 8; ++v) TR[v * T + ci + SS] = f[v];
  }
  const bool moving = __syncthreads_or(mv);
  moved = moving;
  if (late_pf<AXIS>()) prefetch();  // the right states in RSB are consumed

  // ---- P7: Lagrangian update of zones [3, zmax-1] -> LFT -------------------
  // (moving tiles: every cell's conserved state -> FLD for the remap)
  if (live && s < TLv && (moving || (s >= 3 && s <= zmax - 1))) {
    double w[8];
#pragma unroll
    for (int v = 0; v < 8; ++v) w[v] = FLD[fof[v] * T + ci];
    Ops o;
    double cons[8];
    cons[kRho] = w[kRho];
    cons[kUn] = w[kRho] * w[kUn];
    cons[kUt1] = w[kRho] * w[kUt1];
    cons[kUt2] = w[kRho] * w[kUt2];
    cons[kBn] = w[kBn];
    cons[kBt1] = w[kBt1];
    cons[kBt2] = w[kBt2];
    cons[kPE] = strip_energy(w, k, o);
    if (s >= 3 && s <= zmax - 1) {
      const double dx0 = __ldg(A.dx + q);
      const double dxp = dx0 + dt * (CF[ci + SS] - CF[ci]);
      if (!(dxp > 0.0)) {
        atomicMin(s_err, err_key(*A.step, A.phase, AXIS,
                                 (pencil_index() << 20) | ((unsigned long long)q << 2) |
                                     kErrStepRejected));
      } else {
        double u[8];
        const double r_dxp = o.rcp(dxp);
        const double shrink = o.div(dx0, dxp, r_dxp);
#pragma unroll
        for (int v = 0; v < 8; ++v)
          u[v] = cons[v] * shrink -
                 o.div(dt * (TR[v * T + ci + SS] - TR[v * T + ci]), dxp, r_dxp);
        const double internal =
            (u[kPE] - o.dv(0.5 * ((u[kUn] * u[kUn] + u[kUt1] * u[kUt1]) + u[kUt2] * u[kUt2]),
                           u[kRho])) -
            o.div((u[kBn] * u[kBn] + u[kBt1] * u[kBt1]) + u[kBt2] * u[kBt2], c.two_mu0,
                  k.r_two_mu0);
#pragma unroll
        for (int v = 0; v < 8; ++v) LFT[v * T + ci] = u[v];
        if (c.pressure_floor <= 0.0 && (!(u[kRho] > 0.0) || !(internal > 0.0)))
          atomicMin(s_err, err_key(*A.step, A.phase, AXIS,
                                   (pencil_index() << 20) | ((unsigned long long)q << 2) |
                                       kErrLagUnphysical));
      }
    }
    tbad |= o.bad;
    if (moving) {
#pragma unroll
      for (int v = 0; v < 8; ++v) FLD[v * T + ci] = cons[v];
    }
  }
  lsync(2);

  const bool e8 = live && s >= 4 && s <= TLv - 4;
  if (moving) {
    // ---- P7b: conserved slopes at [1, TLv-2] -> TR (fluxes dead) ----------
    if (live && s >= 1 && s <= TLv - 2) {
      const SlopeC sc = slope_coef(A.slope, q);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const double* cv = FLD + v * T + ci;
        TR[v * T + ci] = slope_with(cv[-SS], cv[0], cv[SS], sc);
      }
    }
    lsync(3);
    // ---- P8: slivers at edges [4, TLv-4] --------------------------------
    double sl[8];
#pragma unroll
    for (int v = 0; v < 8; ++v) sl[v] = 0.0;
    if (e8) {
      const double delta = CF[ci] * dt;
      if (delta != 0.0) {
        const bool right = delta > 0.0;
        const int kc = right ? ci - SS : ci;  // upwind zone
        const int kq = right ? q - 1 : q;
        const double width = __ldg(A.dx + kq) + dt * (CF[kc + SS] - CF[kc]);
        double e0[kQfcN], e1[kQfcN];
#pragma unroll
        for (int j = 0; j < kQfcN; ++j) {
          e0[j] = __ldg(A.qfc + kQfcN * kq + j);
          e1[j] = __ldg(A.qfc + kQfcN * (kq + 1) + j);
        }
        Ops o;
        const double sigma = o.dv(right ? delta : -delta, width);
        const double hs = 0.5 * sigma;
        const double tw = tw_of(sigma, k, o);
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const double* cv = FLD + v * T + kc;
          const double* dv = TR + v * T + kc;
          auto win = [&](int j) { return cv[j * SS]; };
          auto dwin = [&](int j) { return dv[j * SS]; };
          double al, ar, six;
          zone_parabola_dm(win, dwin, e0, e1, k, o, al, ar, six);
          const double mean =
              right ? avg_right(al, ar, six, hs, tw) : avg_left(al, ar, six, hs, tw);
          sl[v] = delta * (mean + (LFT[v * T + kc] - cv[0]));
        }
        tbad |= o.bad;
      }
    }
    lsync(4);
    if (e8) {
#pragma unroll
      for (int v = 0; v < 8; ++v) TR[v * T + ci] = sl[v];
    }
    lsync(5);
  }

  // ---- P9: remap, cons_to_prim, store (zones [4, TLv-5]) ------------------
  stored = whole && PPMLR_SWEEP_TMA_STORE;
  if (live && s >= 4 && s <= TLv - 5) {
    const double dxe = __ldg(A.dx + q);
    const double r_dxe = __ldg(A.rdx + q);
    const double width = dxe + dt * (CF[ci + SS] - CF[ci]);
    double out[8], u[8], cs[8];
    Ops o;
    const double scale = o.div(width, dxe, r_dxe);
    if (moving) {
#pragma unroll
      for (int v = 0; v < 8; ++v)
        u[v] = LFT[v * T + ci] * scale + o.div(TR[v * T + ci] - TR[v * T + ci + SS], dxe, r_dxe);
    } else {
#pragma unroll
      for (int v = 0; v < 8; ++v)  // no sliver (strict: the reference's + (0 - 0)/dx)
        u[v] = Ops::kFastMath ? LFT[v * T + ci] * scale
                              : LFT[v * T + ci] * scale + o.div(0.0 - 0.0, dxe, r_dxe);
    }
    cs[0] = u[kRho];
    cs[1 + a] = u[kUn];
    cs[1 + b] = u[kUt1];
    cs[1 + d] = u[kUt2];
    cs[4 + a] = u[kBn];
    cs[4 + b] = u[kBt1];
    cs[4 + d] = u[kBt2];
    cs[7] = u[kPE];
    const int bad = cons_to_prim3(cs, out, k, o);
    tbad |= o.bad;
    if (bad) {
      atomicMin(s_err, err_key(*A.step, A.phase, AXIS,
                               (pencil_index() << 20) | (1ull << 19) |
                                   ((unsigned long long)(q - 4) << 2) |
                                   (bad == 1 ? kErrDensity : kErrPressure)));
    } else if (stored) {
      // dense box order of the L interior zones x NP pencils (FLD is dead)
      const int bi = AXIS == 0 ? p * A.L + (s - 4) : (s - 4) * NP + p;
#pragma unroll
      for (int f = 0; f < 8; ++f) FLD[f * T + bi] = out[f];
    } else {
      const long long off = (long long)(g0 + p + 4) * A.stride_g +
                            (long long)(oc + 4) * A.stride_o + (long long)q * A.stride_a;
#pragma unroll
      for (int f = 0; f < 8; ++f) A.dst[f][off] = out[f];
    }
  }
  if (stored) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  return tbad;
}

// One elected thread: the 8 field boxes of tile `id` into FLD, on `mbar`.
#ifndef PPMLR_SWEEP_V2_BD_L2
#define PPMLR_SWEEP_V2_BD_L2 0  // dipole: B_d boxes prefetched into L2 with the fields (C5: +1.3%, off)
#endif
template <int AXIS, int NP, int TL, bool DIPOLE = false>
__device__ __forceinline__ void tma_load_fields(const SweepArgs& A, const SweepMaps& M,
                                                const TileId id, double* FLD,
                                                unsigned long long* mbar) {
  const int TLr = TL > 0 ? TL : A.L + 8;
  const int T = slot_stride(NP * TLr);
  const unsigned kBox = NP * TLr * sizeof(double);
  const int a0 = id.seg * A.L, g = id.grp * NP + 4, o = id.oc + 4;
  const int cx = AXIS == 0 ? a0 : g;
  const int cy = AXIS == 0 ? g : (AXIS == 1 ? a0 : o);
  const int cz = AXIS == 2 ? a0 : o;
  const unsigned bar = smem_u32(mbar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
               "r"(kBox * 8u)
               : "memory");
#pragma unroll
  for (int f = 0; f < 8; ++f)
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(FLD + f * T)),
        "l"(reinterpret_cast<unsigned long long>(&M.f[f])), "r"(cx), "r"(cy), "r"(cz),
        "r"(bar)
        : "memory");
  if (DIPOLE && PPMLR_SWEEP_V2_BD_L2) {
#pragma unroll
    for (int f = 0; f < 3; ++f)
      asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(
                       reinterpret_cast<unsigned long long>(&M.bd[f])),
                   "r"(cx), "r"(cy), "r"(cz)
                   : "memory");
  }
}

// Tile t of a (part) launch: the split coordinate runs over its part only.
#ifndef PPMLR_SWEEP_Z_GROUPS_FIRST
// z sweeps: claim tiles pencil group (x) first, then y, then the z segment,
// so the CTAs in flight share the same 72 z-planes (page / DRAM-row
// locality) instead of spanning the whole z extent
#define PPMLR_SWEEP_Z_GROUPS_FIRST 1
#endif
#ifndef PPMLR_SWEEP_X_GROUPS_FIRST
// x sweeps: y groups first too -- CTAs in flight share one x segment, so
// its geometry-table entries stay in L1 (the segments' 8-cell halos are
// re-read from DRAM instead): blast +0.3%, C5 +0.5%, strict +0.2%
#define PPMLR_SWEEP_X_GROUPS_FIRST 1
#endif
#ifndef PPMLR_SWEEP_Y_GROUPS_FIRST
#define PPMLR_SWEEP_Y_GROUPS_FIRST 0  // y sweeps too: measured neutral (C5 79.64 vs 79.79 ms)
#endif
template <int AXIS>
__device__ __forceinline__ TileId tile_of_v2(const SweepArgs& A, int t) {
  const int ns = AXIS == 0 ? split_count(A.part, A.cl, A.cr, A.nseg) : A.nseg;
  const int ng = AXIS == 0 ? A.ngroups : split_count(A.part, A.cl, A.cr, A.ngroups);
  if (AXIS == 0 && PPMLR_SWEEP_X_GROUPS_FIRST) {  // y groups, then z, then the segment
    const int rest = t / ng;
    const int v = t - rest * ng, w = rest % A.no;
    return {split_unit(A.part, A.cl, A.cr, rest / A.no), v, w};
  }
  if ((AXIS == 2 && PPMLR_SWEEP_Z_GROUPS_FIRST) || (AXIS == 1 && PPMLR_SWEEP_Y_GROUPS_FIRST)) {
    const int rest = t / ng;
    const int v = t - rest * ng, w = rest % A.no;
    return {rest / A.no, split_unit(A.part, A.cl, A.cr, v), w};
  }
  const int rest = t / ns;
  const int u = t - rest * ns, v = rest % ng;
  return {AXIS == 0 ? split_unit(A.part, A.cl, A.cr, u) : u,
          AXIS == 0 ? v : split_unit(A.part, A.cl, A.cr, v), rest / ng};
}

// Sites (bit j of the mask) whose phase barrier is a neighbour-warp one.
// Measured (fast): P0|P3 + P3|P4 local: C5 sweep -2.7%, blast neutral, C2
// -0.4%; the Lagrangian / remap sites local too: blast +1.5-1.8%.  Strict
// build (right states in registers): C5 +3.5%, blast +2% -- off.
#ifndef PPMLR_SWEEP_V2_LSYNC
#ifdef PPMLR_FAST_MATH
#define PPMLR_SWEEP_V2_LSYNC 3
#else
#define PPMLR_SWEEP_V2_LSYNC 0
#endif
#endif
#ifndef PPMLR_SWEEP_V2_MINB
#define PPMLR_SWEEP_V2_MINB 3
#endif
#ifndef PPMLR_SWEEP_V2_DYN
#define PPMLR_SWEEP_V2_DYN 1  // tiles beyond the first wave claimed from a counter
#endif

// Persistent main instance (grid = min(tiles, resident CTAs)); flagged
// tiles go to the EXACT instance of sweep.cuh as before.  Each CTA starts
// on tile blockIdx.x; the elected thread claims the next tile (a global
// counter, so tiles with a moving edge — dearer — balance across CTAs)
// when the current one starts and prefetches its fields.
template <int AXIS, bool DIPOLE, int NP, int TL>
__global__ void __launch_bounds__(NP*(TL > 0 ? TL : kSweepTL), PPMLR_SWEEP_V2_MINB)
    sweep_kernel_v2(const SweepArgs A, const __grid_constant__ SweepMaps M) {
  extern __shared__ __align__(128) double smem[];
  __shared__ unsigned long long s_err;
  __shared__ __align__(8) unsigned long long s_mbar[2];
  // neighbour-warp phase barriers (PPMLR_SWEEP_V2_LSYNC): one mbarrier per
  // warp and sync site (sites 0-2 every tile, 3-5 moving tiles only), plus
  // the "previous result box read" signal that gates the RSB writes of P3
  constexpr int kNW = TL > 0 ? NP * TL / 32 : 1;
  constexpr bool kLocal = PPMLR_SWEEP_V2_LSYNC && TL > 0 && (NP * TL) % 32 == 0;
  __shared__ __align__(8) unsigned long long s_lbar[kLocal ? 6 * kNW : 1];
  __shared__ __align__(8) unsigned long long s_drain;
  __shared__ unsigned s_nmov;
  // the claimed tile of each buffer, decoded once by the elected thread:
  // {t, seg, grp, oc}
  __shared__ int s_tile[2][4];
  const int T = slot_stride(NP * (TL > 0 ? TL : A.L + 8));
  const int ntiles = (AXIS == 0 ? split_count(A.part, A.cl, A.cr, A.nseg) : A.nseg) *
                     (AXIS == 0 ? A.ngroups : split_count(A.part, A.cl, A.cr, A.ngroups)) * A.no;
  auto claim = [&](int slot, int t) {  // elected thread
    const TileId id = tile_of_v2<AXIS>(A, t < ntiles ? t : 0);
    s_tile[slot][0] = t;
    s_tile[slot][1] = id.seg;
    s_tile[slot][2] = id.grp;
    s_tile[slot][3] = id.oc;
    return id;
  };
  if (threadIdx.x == 0) {
    s_err = kNoError;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_mbar[0])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_mbar[1])) : "memory");
    if (kLocal) {
      for (int j = 0; j < 6 * kNW; ++j)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(smem_u32(&s_lbar[j]))
                     : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_drain)) : "memory");
      s_nmov = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const TileId id0 = claim(0, blockIdx.x);
    if ((int)blockIdx.x < ntiles) tma_load_fields<AXIS, NP, TL, DIPOLE>(A, M, id0, smem, &s_mbar[0]);
  }
  __syncthreads();
#pragma unroll 1
  for (int i = 0;; ++i) {
    const int buf = i & 1;
    const int t = s_tile[buf][0];
    if (t >= ntiles) break;
    double* FLD = smem + buf * 8 * T;
    const TileId id = {s_tile[buf][1], s_tile[buf][2], s_tile[buf][3]};
    double* NXT = smem + (buf ^ 1) * 8 * T;
    int tn = 0;
    TileId idn{0, 0, 0};
    if (threadIdx.x == 0) {
      tn = PPMLR_SWEEP_V2_DYN ? (int)gridDim.x + (int)atomicAdd(A.tile_ctr, 1u)
                              : t + (int)gridDim.x;
      idn = claim(buf ^ 1, tn);
      // the other buffer held the previous tile's result box: its TMA store
      // must have read it before it is reused (scratch, then the next fields)
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      if (kLocal)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&s_drain))
                     : "memory");
    }
    // Phase barrier j of the tile: with kLocal, warp w waits only for warps
    // w-1 and w+1 (every smem dependency of a phase on the one before spans
    // at most 2 strip positions = one neighbouring warp; the staged result
    // box of P9 lands at most 28 threads back, outside what warp w-2 reads)
    auto lsync = [&](int j) {
      if (!kLocal || !((PPMLR_SWEEP_V2_LSYNC >> j) & 1)) {
        __syncthreads();
        return;
      }
      const int w = threadIdx.x >> 5;
      const unsigned par = j < 3 ? (unsigned)i & 1u : s_nmov & 1u;
      unsigned long long* b = s_lbar + j * kNW;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b + w)) : "memory");
      __syncwarp();
      if (j == 0 && rs_of<AXIS>()) mbar_wait(&s_drain, (unsigned)i & 1u);
      if (w > 0) mbar_wait(b + w - 1, par);
      if (w + 1 < kNW) mbar_wait(b + w + 1, par);
    };
    auto prefetch = [&]() {
      if (threadIdx.x == 0 && tn < ntiles) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tma_load_fields<AXIS, NP, TL, DIPOLE>(A, M, idn, NXT, &s_mbar[buf ^ 1]);
      }
    };
    if (!late_pf<AXIS>()) prefetch();
    mbar_wait(&s_mbar[buf], (unsigned)(i >> 1) & 1u);
    bool stored = false;
    bool moved = false;
    const bool bad = sweep_tile_v2<AXIS, DIPOLE, NP, TL, MainOps>(A, M, id, smem, FLD, NXT,
                                                                  &s_err, stored, prefetch, lsync,
                                                                  moved);
    const bool any_bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) {
      if (kLocal && moved) ++s_nmov;
      if (stored) {
        const int a0 = id.seg * A.L + 4, g = id.grp * NP + 4, o = id.oc + 4;
        const int c0 = AXIS == 0 ? a0 : g;
        const int c1 = AXIS == 0 ? g : (AXIS == 1 ? a0 : o);
        const int c2 = AXIS == 2 ? a0 : o;
#pragma unroll
        for (int f = 0; f < 8; ++f)
          asm volatile(
              "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                  reinterpret_cast<unsigned long long>(&M.out[f])),
              "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(FLD + f * T))
              : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      if (any_bad)  // the tile's full-grid index (sweep.cuh tile_of)
        A.redo_list[atomicAdd(A.redo_count, 1u)] = id.seg + A.nseg * (id.grp + A.ngroups * id.oc);
      else if (s_err != kNoError)
        atomicMin(A.err, s_err);
      s_err = kNoError;
    }
  }
  // the shared memory must outlive the last stores' reads of it
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

}  // namespace PPMLR_KNS
}  // namespace ppmlr_b200
