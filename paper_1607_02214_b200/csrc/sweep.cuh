// Directional PPMLR sweep kernel (sm_100a, FP64): the whole of the
// reference's sweep_axis -> sweep_1d (proj/src/stepper.cpp:249-282,
// proj/src/ppm1d.cpp:111-364) for every pencil of one block along AXIS.
//
// Work decomposition.  A CTA owns a tile of NP = 4 adjacent pencils x one
// segment of TL = L + 8 strip positions (L interior cells plus the 4-cell
// dependency halo on each side), one cell per thread.  One
// elected thread streams the tile in with TMA (one box per field plane,
// completing on an mbarrier); the tile is staged in shared memory,
// structure-of-arrays, and the 1-D algorithm runs as cell-parallel phases
// separated by __syncthreads():
//
//   P0  strip-frame prim, cons, c_f from the TMA'd fields       -> PRIM, CONS, CF
//       (fast XS: primitive slopes here too -> TR; PRIM left unwritten, P3
//       reads the field slots and PRIM/SA swap roles from P4 on)
//   P1  primitive slopes (once per cell)                        -> SA
//   P2  (edge-once schedule) interface value per edge           -> TR
//   P3  per zone: interface values, limited parabola, traced
//       edge states                                             -> PRIM:=R, SA|TR:=L
//   P4  per edge: Lagrangian Riemann solve                      -> CF:=u*, SA:=flux
//   P7  per zone: Lagrangian update + the reference's checks    -> PRIM:=lag
//   P7b tiles with a moving edge: conserved slopes per cell     -> SA|TR
//       (XS: in P7's phase, the tile's vote taken at P4's barrier)
//   P8  per moving edge only: the upwind zone's conserved
//       parabola and the remap sliver                           -> CONS|SA:=sliver
//   P9  per zone: remap onto the fixed mesh, cons_to_prim; whole
//       tiles leave through TMA box stores, partial ones per thread
//
// Shared FP64 slots per cell: 25 (+3 with the dipole) = 57.6 KB for the
// 288-cell tile, or 33 (the extra-slot schedule XS: TR) = 76 KB; 3 CTAs per
// SM at <= 72 registers either way.  XS lets the traced left states and the
// slivers skip a write-after-read barrier; its edge-once variant (EO,
// strict build) computes each interface value once.  Results are
// bit-identical to the reference in the strict build: every output is
// produced by the reference's own expression sequence; the reorganisations
// are exact (hoisted geometry, interface values / slivers / sigma terms
// evaluated once per edge instead of twice, conserved slopes per cell only
// where the tile moves, segment halos recomputed).  Arithmetic goes through
// an Ops policy (exact_div.cuh): the main instance runs branch-free fast
// paths and flags tiles whose guards failed; the EXACT instance re-runs
// those tiles with plain `/` and `sqrt`.
#pragma once
#include <cuda.h>  // CUtensorMap (the maps are encoded on the host, block.cu)

#include "grid_types.cuh"
#include "ppmlr_dev.cuh"

namespace ppmlr_b200 {

// Compile-time tile of the main sweep instantiation (default L = 64 interior
// cells per segment, 4 pencils per tile).
#ifndef PPMLR_SWEEP_NP
#define PPMLR_SWEEP_NP 4   // pencils per tile
#endif
#ifndef PPMLR_SWEEP_TL
#define PPMLR_SWEEP_TL 72  // strip positions per tile (L + 8; even)
#endif
#ifndef PPMLR_SWEEP_TL2
#define PPMLR_SWEEP_TL2 64  // second compile-time tile (L = 56) for axes < 256 cells
#endif
constexpr int kSweepNP = PPMLR_SWEEP_NP;
constexpr int kSweepTL = PPMLR_SWEEP_TL;
constexpr int kSweepTL2 = PPMLR_SWEEP_TL2;
#ifndef PPMLR_SWEEP_MINB
#define PPMLR_SWEEP_MINB 3  // resident CTAs per SM the register budget targets
#endif
#ifndef PPMLR_SWEEP_TMA
#define PPMLR_SWEEP_TMA 1  // TMA tile loads for the compile-time tile
#endif
#ifndef PPMLR_SWEEP_TMA_STORE
#define PPMLR_SWEEP_TMA_STORE 1  // TMA stores of whole tiles' results
#endif
#ifndef PPMLR_SWEEP_XSLOTS
#define PPMLR_SWEEP_XSLOTS 1  // 8 more slots without the dipole: 2 fewer barriers
#endif
// the extra-slot schedule with the dipole, per build
#ifndef PPMLR_SWEEP_XSD_FAST
#define PPMLR_SWEEP_XSD_FAST 0    // measured -2.7% (P4's global dipole loads)
#endif
#ifndef PPMLR_SWEEP_XSD_STRICT
#define PPMLR_SWEEP_XSD_STRICT 1  // enables the edge-once trace (+0.5%)
#endif
#ifdef PPMLR_FAST_MATH
#define PPMLR_SWEEP_XSLOTS_DIPOLE PPMLR_SWEEP_XSD_FAST
#else
#define PPMLR_SWEEP_XSLOTS_DIPOLE PPMLR_SWEEP_XSD_STRICT
#endif
#ifndef PPMLR_SWEEP_EDGE_ONCE
#ifdef PPMLR_FAST_MATH
#define PPMLR_SWEEP_EDGE_ONCE 0  // measured: a wash in the fast build (more smem traffic)
#else
#define PPMLR_SWEEP_EDGE_ONCE 1  // strict build: interface values once per edge (+3%)
#endif
#endif
#ifndef PPMLR_SWEEP_CSLOPE
#define PPMLR_SWEEP_CSLOPE 1  // conserved slopes once per cell (P7b) vs per moving edge
#endif
#ifndef PPMLR_SWEEP_FUSE01
// XS schedule with TMA'd tiles: the primitive slopes are taken in P0 from the
// TMA'd input slots (the strip-frame primitives are a permutation of the
// fields), into TR; P3 then writes the traced left states into SA.  One
// barrier fewer per tile.
#define PPMLR_SWEEP_FUSE01 1
#endif
#ifndef PPMLR_SWEEP_P0NOPRIM
// F01: P0 leaves PRIM unwritten (the TMA'd field slots in SA already hold
// the primitives, permuted); P3 reads them there, writes the traced left
// states to PRIM at once and the right states to SA after its barrier, and
// from P4 on the two regions swap roles.
#define PPMLR_SWEEP_P0NOPRIM 1
#endif
#ifndef PPMLR_SWEEP_FUSE7B
// extra-slot schedules: the tile's "any moving edge" vote is taken at P4's
// closing barrier, the conserved slopes (P7b) are computed in P7's phase into
// the dead TR slots, and the slivers go to SA (fluxes dead after P7).  One
// barrier fewer per moving tile (blast 512^3 sweep: fast 11.21 -> 11.07 ms,
// strict 15.36 -> 15.30).
#define PPMLR_SWEEP_FUSE7B 1
#endif

// TMA descriptors of the sweep's input: the 8 field planes of the source
// buffer and the 3 dipole planes, each a 3-D (x, y, z) tensor over the padded
// ghost-inclusive block with the tile box of this axis ({72,4,1} for x,
// {4,72,1} for y, {4,1,72} for z; TL = L + 8 of the block's axis in
// place of 72 for the runtime tile).  The box lands in shared memory in
// exactly the tile's cell order (ci), one field per slot.
struct SweepMaps {
  CUtensorMap f[8];
  CUtensorMap bd[3];
  CUtensorMap out[8];  // destination planes, box of the L interior zones
};

struct SweepArgs {
  const double* src[8];  // field planes of the input buffer (padded block layout)
  double* dst[8];        // field planes of the output buffer
  const double* bd[3];   // dipole planes (DIPOLE only)
  const double* dx;      // ghost-inclusive spacings along AXIS (span entries)
  const double* rdx;     // rcp_refined(dx) per position (exact-division helper)
  const double* slope;   // 3 per strip position: c0, A, B
  const double* qfc;     // 5 per edge index m: e0..e4
  long long stride_a, stride_g, stride_o;  // element strides: sweep / group / other axis
  int n;                 // interior cells along AXIS
  int ng, no;            // interior cells along the group / other axis
  int nb;                // interior cells along (AXIS+1)%3 (reference pencil order)
  int L;                 // interior cells per segment (TL = L + 8)
  int nseg, ngroups;
  const double* dt;      // device scalar
  unsigned long long* err;
  const unsigned long long* step;  // device step counter for error keys
  int phase;             // kPhaseSweep{0,1,2}
  Consts c;
  unsigned* redo_count;  // tiles whose fast-path guards failed ...
  unsigned* redo_list;   // ... are re-run exactly by the EXACT instance
  unsigned* tile_ctr;    // persistent schedule (sweep_v2.cuh): tiles claimed so far
  // Split launches for the halo overlap (dist.py): the tiles' x coordinate
  // unit (the segment of an x sweep, the pencil group of a y/z sweep) is
  // "boundary" in [0, cl) and [cr, count) -- it holds one of the 4 x cells
  // a neighbour needs -- and "interior" in [cl, cr).  part 0: every tile,
  // 1: boundary units only, 2: interior units only.
  int part, cl, cr;
  // y / z sweeps with the dipole: B_d in bricks along the sweep axis
  // (block.cu bd_bricks_kernel): component c, interior index o of the other
  // axis, x group xg (4 cells from x = 4), strip position q, pencil p at
  // bdz[c * bdz_cs + ((o * bdz_ngx + xg) * bdz_s2 + q) * 4 + p] -- a tile's
  // 72 x 4 values are one contiguous 2.3 KB run instead of 72 rows of 32 B
  // (z: 72 planes, i.e. 2 MB pages, apart)
  const double* bdz;
  long long bdz_cs;
  int bdz_ngx, bdz_s2;
};


namespace PPMLR_KNS {

// Strided view of one cell's 8 strip variables in shared memory.
struct SmemVec {
  const double* p;
  int stride;
  __device__ __forceinline__ double operator[](int v) const { return p[v * stride]; }
};

template <int AXIS>
struct AxisMap {
  // group axis (pencils adjacent in memory for y/z sweeps), other axis
  static constexpr int G = AXIS == 0 ? 1 : 0;
  static constexpr int O = AXIS == 2 ? 1 : 2;
  static constexpr int B = (AXIS + 1) % 3;  // reference t1 axis
};

template <bool B>
struct FlatTag {
  static constexpr bool value = B;
};

// Tile coordinates: segment along AXIS, group of NP pencils, other axis.
struct TileId {
  int seg, grp, oc;
};
__device__ __forceinline__ TileId tile_of(const SweepArgs& A, int t) {
  const int rest = t / A.nseg;
  return {t - rest * A.nseg, rest % A.ngroups, rest / A.ngroups};
}

// The limited parabola of zone (tile row s) from the 5-point window of one
// variable: reconstruct() (ppm1d.cpp:200-247) restricted to one zone.
template <class W, class Ops>
__device__ __forceinline__ void zone_parabola(const W& q, const SlopeC* sc, const double* e0,
                                              const double* e1, const KC& k, Ops& o,
                                              double& al, double& ar, double& six) {
  // q(-2..2); sc: slope coefficients at positions q-1, q, q+1 (3 each)
  const double dmm = slope_with(q(-2), q(-1), q(0), sc[0]);
  const double dm0 = slope_with(q(-1), q(0), q(1), sc[1]);
  const double dmp = slope_with(q(0), q(1), q(2), sc[2]);
  al = iface(q(-1), q(0), dmm, dm0, e0);
  ar = iface(q(0), q(1), dm0, dmp, e1);
  limit_parabola(al, ar, q(0), six, k, o);
}

// Limited parabola of a zone from its 3-point window and the stored slopes
// of the window (reconstruct(), ppm1d.cpp:200-247, restricted to one zone).
template <class W, class D, class Ops>
__device__ __forceinline__ void zone_parabola_dm(const W& q, const D& dm, const double* e0,
                                                 const double* e1, const KC& k, Ops& o,
                                                 double& al, double& ar, double& six) {
  al = iface(q(-1), q(0), dm(-1), dm(0), e0);
  ar = iface(q(0), q(1), dm(0), dm(1), e1);
  limit_parabola(al, ar, q(0), six, k, o);
}

// The two traced edge states of a zone (P3) from its 3-point window and the
// stored slopes: the fast build takes the fused limiter (traced_lr).
template <class W, class D, class Ops>
__device__ __forceinline__ void zone_traced_dm(const W& q, const D& dm, const double* e0,
                                               const double* e1, const KC& k, Ops& o,
                                               double hs, double tw, double& l, double& r) {
#if defined(PPMLR_FAST_MATH) && PPMLR_FAST_TRACED
  const double al = iface(q(-1), q(0), dm(-1), dm(0), e0);
  const double ar = iface(q(0), q(1), dm(0), dm(1), e1);
  traced_lr(al, ar, q(0), hs, tw, k.r3, l, r);
#else
  double al, ar, six;
  zone_parabola_dm(q, dm, e0, e1, k, o, al, ar, six);
  l = avg_left(al, ar, six, hs, tw);
  r = avg_right(al, ar, six, hs, tw);
#endif
}

// Shared slots start on 128-byte boundaries (the TMA destination rule).
__host__ __device__ constexpr int slot_stride(int cells) { return (cells + 15) & ~15; }

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

// One elected thread: expect the tile's bytes on `mbar` and issue the TMA
// loads of the 8 fields (+3 dipole planes) into SA / BD.
template <int AXIS, bool DIPOLE, int NP, int TLC>
__device__ __forceinline__ void tma_load_tile(const SweepArgs& A, const SweepMaps& M, int seg,
                                              int grp, int oc, double* smem,
                                              unsigned long long* mbar) {
  const int NT = NP * (TLC > 0 ? TLC : A.L + 8);
  const int T = slot_stride(NT);
  const unsigned kBox = NT * sizeof(double);
  const int a0 = seg * A.L, g = grp * NP + 4, o = oc + 4;
  const int cx = AXIS == 0 ? a0 : g;
  const int cy = AXIS == 0 ? g : (AXIS == 1 ? a0 : o);
  const int cz = AXIS == 2 ? a0 : o;
  const unsigned bar = smem_u32(mbar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
               "r"(kBox * (DIPOLE ? 11u : 8u))
               : "memory");
  double* SA = smem + 17 * T;
  double* BD = smem + 25 * T;
#pragma unroll
  for (int f = 0; f < 8 + (DIPOLE ? 3 : 0); ++f) {
    const CUtensorMap* m = f < 8 ? &M.f[f] : &M.bd[f - 8];
    double* dst = f < 8 ? SA + f * T : BD + (f - 8) * T;
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(m)), "r"(cx), "r"(cy), "r"(cz), "r"(bar)
        : "memory");
  }
}

__device__ __forceinline__ void mbar_wait(unsigned long long* mbar, unsigned parity) {
  const unsigned bar = smem_u32(mbar);
  unsigned done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.b32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
}

// TMA: the tile's inputs arrive in SA / BD through tma_load_tile (issued by
// the caller, completing on `mbar`) instead of per-thread global loads.
template <int AXIS, bool DIPOLE, int NP, int TLC, class Ops, bool TMA = false>
__device__ __forceinline__ bool sweep_tile(const SweepArgs& A, const int seg, const int grp,
                                           const int oc, double* smem,
                                           unsigned long long* s_err,
                                           unsigned long long* mbar = nullptr,
                                           int* store = nullptr) {
  bool tbad = false;
  const int TL = TLC > 0 ? TLC : A.L + 8;
  const int NT = NP * TL;          // cells of the tile
  const int T = slot_stride(NT);   // doubles per shared slot (128 B multiple)
  double* PRIM = smem;
  double* CONS = smem + 8 * T;
  double* CF = smem + 16 * T;
  double* SA = smem + 17 * T;
  double* BD = smem + 25 * T;
  // XS (no dipole, 33 slots): traced left states and later the slivers get
  // their own slots TR, so neither waits for a write-after-read barrier
  // With the dipole too: its three planes land in TR[0..2] (the same slots
  // the BD region would take), P0 reads them, and P4 takes the two cells'
  // dipole from global memory (L2) instead of a shared BD region.
  constexpr bool XS = PPMLR_SWEEP_XSLOTS && (!DIPOLE || PPMLR_SWEEP_XSLOTS_DIPOLE);
  double* TR = smem + 25 * T;
  constexpr bool F01 = PPMLR_SWEEP_FUSE01 && TMA && XS && !(XS && PPMLR_SWEEP_EDGE_ONCE);
  // F01: slopes in TR, the traced left states in SA
  constexpr bool NP0 = F01 && PPMLR_SWEEP_P0NOPRIM;
  double* SLP = F01 ? TR : SA;
  double* LFT = NP0 ? PRIM : (F01 ? SA : TR);
  const int SS = AXIS == 0 ? 1 : NP;
  // (with the dipole, measured -0.4% on the strict magnetosphere: kept off)
  constexpr bool F7 = PPMLR_SWEEP_FUSE7B && XS && !DIPOLE && PPMLR_SWEEP_CSLOPE;

  const int nn = A.n + 8;
  const int seg0 = seg * A.L;
  const int TLv = min(TL, nn - seg0);
  // TMA store of the results only for whole tiles (a partial box would
  // write ghost or padding cells)
  const bool final_seg = seg == A.nseg - 1;
  const int zmax = final_seg ? TLv - 2 : TL - 3;
  const int g0 = grp * NP;
  const int npv = min(NP, A.ng - g0);
  const bool tma_store = TMA && PPMLR_SWEEP_TMA_STORE && TLv == TL && npv == NP;
  const double dt = *A.dt;
  const Consts& c = A.c;
  const KC k = make_kc(c);
  const long long base = (long long)(g0 + 4) * A.stride_g + (long long)(oc + 4) * A.stride_o +
                         (long long)seg0 * A.stride_a;
  // one cell per thread (the launcher guarantees blockDim.x >= T)
  const int ci = threadIdx.x;
  int s, p;
  if (AXIS == 0) {
    p = ci / TL;
    s = ci - p * TL;
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
  // field slot of each strip variable (the TMA'd fields are in field order)
  constexpr int fof[8] = {0, 1 + a, 1 + b, 1 + d, 4 + a, 4 + b, 4 + d, 7};

  // ---- P0 ---------------------------------------------------------------
  if (TMA) mbar_wait(mbar, 0);
  if (live && s < TLv) {
    const long long off = base + (long long)p * A.stride_g + (long long)s * A.stride_a;
    double qv[8];
#pragma unroll
    for (int f = 0; f < 8; ++f) qv[f] = TMA ? SA[f * T + ci] : __ldg(A.src[f] + off);
    double b0 = 0.0, b1 = 0.0, b2 = 0.0;
    if (DIPOLE) {
      b0 = TMA ? BD[ci] : __ldg(A.bd[0] + off);
      b1 = TMA ? BD[T + ci] : __ldg(A.bd[1] + off);
      b2 = TMA ? BD[2 * T + ci] : __ldg(A.bd[2] + off);
      if (!XS) {
        BD[0 * T + ci] = AXIS == 0 ? b0 : (AXIS == 1 ? b1 : b2);
        BD[1 * T + ci] = AXIS == 0 ? b1 : (AXIS == 1 ? b2 : b0);
        BD[2 * T + ci] = AXIS == 0 ? b2 : (AXIS == 1 ? b0 : b1);
      }
    }
    double w[8];
    w[kRho] = qv[0];
    w[kUn] = qv[1 + a];
    w[kUt1] = qv[1 + b];
    w[kUt2] = qv[1 + d];
    w[kBn] = qv[4 + a];
    w[kBt1] = qv[4 + b];
    w[kBt2] = qv[4 + d];
    w[kPE] = qv[7];
    Ops o;
    const double cf = fast_speed3<AXIS>(qv, b0, b1, b2, k, o);
    const double e = strip_energy(w, k, o);
    tbad |= o.bad;
    CF[ci] = cf;
    if (!NP0) {
#pragma unroll
      for (int v = 0; v < 8; ++v) PRIM[v * T + ci] = w[v];
    }
    CONS[kRho * T + ci] = w[kRho];
    CONS[kUn * T + ci] = w[kRho] * w[kUn];
    CONS[kUt1 * T + ci] = w[kRho] * w[kUt1];
    CONS[kUt2 * T + ci] = w[kRho] * w[kUt2];
    CONS[kBn * T + ci] = w[kBn];
    CONS[kBt1 * T + ci] = w[kBt1];
    CONS[kBt2 * T + ci] = w[kBt2];
    CONS[kPE * T + ci] = e;
    if (F01 && s >= 1 && s <= TLv - 2) {
      // P1 fused: the neighbours' strip-frame primitives straight from the
      // TMA'd fields (PRIM is a pure permutation of them) -> TR
      const SlopeC sc = slope_coef(A.slope, q);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const double* pv = SA + fof[v] * T + ci;
        TR[v * T + ci] = slope_with(pv[-SS], w[v], pv[SS], sc);
      }
    }
  }
  __syncthreads();

  // ---- P1: primitive slopes at s in [1, TLv-2] -> SA ---------------------
  if (!F01 && live && s >= 1 && s <= TLv - 2) {
    const SlopeC sc = slope_coef(A.slope, q);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const double* pv = PRIM + v * T + ci;
      SA[v * T + ci] = slope_with(pv[-SS], pv[0], pv[SS], sc);
    }
  }
  if (!F01) __syncthreads();

  // ---- P3: prim parabolas -> traced states (zones [2, zmax]) ------------
  // ---- P2 (without the dipole): the CW84 interface value of every zone's
  // right edge, once per edge (zone s+1 reads it as its left edge) -> TR
  const bool z3 = live && s >= 2 && s <= zmax;
  const bool flat = q >= nn - 2;  // q >= 2 always here
  constexpr bool EO = XS && PPMLR_SWEEP_EDGE_ONCE;
  if (EO) {
    if (live && s >= 1 && s <= zmax && q <= nn - 3) {
      double e[kQfcN];
#pragma unroll
      for (int j = 0; j < kQfcN; ++j) e[j] = __ldg(A.qfc + kQfcN * (q + 1) + j);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const double* pv = PRIM + v * T + ci;
        const double* dv = SA + v * T + ci;
        TR[v * T + ci] = iface(pv[0], pv[SS], dv[0], dv[SS], e);
      }
    }
    __syncthreads();
    // ---- P3: limiter + traced states per zone from its two edge values;
    // every read is the zone's own (PRIM, TR of s and s-1), so L goes to SA
    // and R to PRIM at once, with no write-after-read barrier
    if (z3) {
      Ops o;
      const double sigma =
          sclamp(o.div(CF[ci] * dt, __ldg(A.dx + q), __ldg(A.rdx + q)), 0.0, 1.0);
      const double hs = 0.5 * sigma;
      const double tw = tw_of(sigma, k, o);
      // the fast build decides the flat strip-end zones once per zone
#ifdef PPMLR_FAST_MATH
      constexpr bool kUnswitchX = true;
#else
      constexpr bool kUnswitchX = false;
#endif
      auto tr = [&](auto F, const int v, double& l, double& r) {
        const double av = PRIM[v * T + ci];
        double al = av, ar = av, six = 0.0;
        if (!decltype(F)::value && (kUnswitchX || !flat)) {
          al = TR[v * T + ci - SS];
          ar = TR[v * T + ci];
          limit_parabola(al, ar, av, six, k, o);
        }
        l = avg_left(al, ar, six, hs, tw);
        r = avg_right(al, ar, six, hs, tw);
      };
      auto all8 = [&](auto F) {
        // rho and p first: they decide the reference's fallback for all eight
        double Lr, Rr, Lp, Rp;
        tr(F, kRho, Lr, Rr);
        tr(F, kPE, Lp, Rp);
        const bool badL = !(Lr > 0.0) || !(Lp > 0.0);
        const bool badR = !(Rr > 0.0) || !(Rp > 0.0);
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          double l, r;
          if (v == kRho) {
            l = Lr;
            r = Rr;
          } else if (v == kPE) {
            l = Lp;
            r = Rp;
          } else {
            tr(F, v, l, r);
          }
          const double own = PRIM[v * T + ci];
          SA[v * T + ci] = badL ? own : l;
          PRIM[v * T + ci] = badR ? own : r;
        }
      };
      if (kUnswitchX && flat)
        all8(FlatTag<true>{});
      else
        all8(FlatTag<false>{});
      tbad |= o.bad;
    }
    __syncthreads();
  } else {
  // ---- P3: prim parabolas -> traced states (zones [2, zmax]) ------------
  // Two halves of four variables, each written back after a barrier, so
  // that only eight traced values are held across a barrier.  The first
  // half holds rho and p, which decide the reference's fallback to the
  // zone's own state for all eight.
  double e0[kQfcN], e1[kQfcN], hs = 0.0, tw = 0.0;
  bool badL = false, badR = false;
  Ops o3;
  if (z3) {
    if (!flat) {
#pragma unroll
      for (int j = 0; j < kQfcN; ++j) {
        e0[j] = __ldg(A.qfc + kQfcN * q + j);
        e1[j] = __ldg(A.qfc + kQfcN * (q + 1) + j);
      }
    }
    const double sigma =
        sclamp(o3.div(CF[ci] * dt, __ldg(A.dx + q), __ldg(A.rdx + q)), 0.0, 1.0);
    hs = 0.5 * sigma;
    tw = tw_of(sigma, k, o3);
  }
  // The strip's last two zones are flat.  The fast build decides that once
  // per zone outside the variable loops (compile-time F); the strict build
  // keeps the test per variable (unswitching costs it registers).
#ifdef PPMLR_FAST_MATH
  constexpr bool kUnswitch = true;
#else
  constexpr bool kUnswitch = false;
#endif
  auto trace = [&](auto F, const int v, double& l, double& r) {
    const double* pv = NP0 ? SA + fof[v] * T + ci : PRIM + v * T + ci;
    const double av = pv[0];
    if (!decltype(F)::value && (kUnswitch || !flat)) {
      const double* dv = SLP + v * T + ci;
      auto win = [&](int j) { return pv[j * SS]; };
      auto dwin = [&](int j) { return dv[j * SS]; };
      zone_traced_dm(win, dwin, e0, e1, k, o3, hs, tw, l, r);
    } else {
      l = avg_left(av, av, 0.0, hs, tw);
      r = avg_right(av, av, 0.0, hs, tw);
    }
  };
  {
  if (XS) {
    // rho and p first (they decide the fallback), then every variable:
    // L straight into TR, R held and written after one barrier
    double R[8];
    auto all8 = [&](auto F) {
      double Lr, Lp;
      trace(F, kRho, Lr, R[kRho]);
      trace(F, kPE, Lp, R[kPE]);
      badL = !(Lr > 0.0) || !(Lp > 0.0);
      badR = !(R[kRho] > 0.0) || !(R[kPE] > 0.0);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        double l = v == kRho ? Lr : Lp;
        if (v != kRho && v != kPE) trace(F, v, l, R[v]);
        LFT[v * T + ci] = l;
      }
      if (badL || badR) {  // rare: the zone falls back to its own state
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          // PRIM (NP0: SA) is rewritten after the barrier
          const double own = NP0 ? SA[fof[v] * T + ci] : PRIM[v * T + ci];
          if (badL) LFT[v * T + ci] = own;
          if (badR) R[v] = own;
        }
      }
    };
    if (z3) {
      if (kUnswitch && flat)
        all8(FlatTag<true>{});
      else
        all8(FlatTag<false>{});
      tbad |= o3.bad;
    }
    __syncthreads();
    if (z3) {
#pragma unroll
      for (int v = 0; v < 8; ++v) (NP0 ? SA : PRIM)[v * T + ci] = R[v];
    }
    if (NP0) {  // from P4 on: right states (then lag values) in SA's slots
      double* t = PRIM;
      PRIM = SA;
      SA = t;
      LFT = SA;
    }
  } else {
  {
    const int H[4] = {kRho, kPE, kUn, kUt1};
    double L[4], R[4];
    if (z3) {
      if (kUnswitch && flat) {
#pragma unroll
        for (int j = 0; j < 4; ++j) trace(FlatTag<true>{}, H[j], L[j], R[j]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) trace(FlatTag<false>{}, H[j], L[j], R[j]);
      }
      badL = !(L[0] > 0.0) || !(L[1] > 0.0);
      badR = !(R[0] > 0.0) || !(R[1] > 0.0);
      if (badL || badR) {  // rare: the zone falls back to its own state
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double own = PRIM[H[j] * T + ci];
          if (badL) L[j] = own;
          if (badR) R[j] = own;
        }
      }
    }
    __syncthreads();
    if (z3) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        PRIM[H[j] * T + ci] = R[j];
        SA[H[j] * T + ci] = L[j];
      }
    }
  }
  {
    const int H[4] = {kUt2, kBn, kBt1, kBt2};
    double L[4], R[4];
    if (z3) {
      if (kUnswitch && flat) {
#pragma unroll
        for (int j = 0; j < 4; ++j) trace(FlatTag<true>{}, H[j], L[j], R[j]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) trace(FlatTag<false>{}, H[j], L[j], R[j]);
      }
      if (badL || badR) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double own = PRIM[H[j] * T + ci];
          if (badL) L[j] = own;
          if (badR) R[j] = own;
        }
      }
      tbad |= o3.bad;
    }
    __syncthreads();
    if (z3) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        PRIM[H[j] * T + ci] = R[j];
        SA[H[j] * T + ci] = L[j];
      }
    }
  }
  }
  __syncthreads();

  }
  }

  // ---- P4: edge solve at m in [3, zmax] ---------------------------------
  bool mv = false;  // F7: a moving edge of P8's range (s in [4, TLv-4])
  if (live && s >= 3 && s <= zmax) {
    double f[8], bl[3] = {0.0, 0.0, 0.0}, br[3] = {0.0, 0.0, 0.0};
    // traced left states: TR in the fast extra-slot schedule, else SA
    const SmemVec ql{PRIM + ci - SS, T}, qr{((XS && !EO) ? LFT : SA) + ci, T};
    if (DIPOLE && XS) {  // strip order (a, b, d) of the zones either side
      const long long off = base + (long long)p * A.stride_g + (long long)s * A.stride_a;
      constexpr int ja = AXIS, jb = (AXIS + 1) % 3, jd = (AXIS + 2) % 3;
      br[0] = __ldg(A.bd[ja] + off);
      br[1] = __ldg(A.bd[jb] + off);
      br[2] = __ldg(A.bd[jd] + off);
      bl[0] = __ldg(A.bd[ja] + off - A.stride_a);
      bl[1] = __ldg(A.bd[jb] + off - A.stride_a);
      bl[2] = __ldg(A.bd[jd] + off - A.stride_a);
    } else if (DIPOLE) {
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        bl[j] = BD[j * T + ci - SS];
        br[j] = BD[j * T + ci];
      }
    }
    Ops o;
    const double us = solve_edge(ql, qr, bl, br, k, f, o);
    tbad |= o.bad;
    CF[ci] = us;
    mv = s >= 4 && s <= TLv - 4 && us * dt != 0.0;
#pragma unroll
    for (int v = 0; v < 8; ++v) SA[v * T + ci] = f[v];
  }
  bool moving = false;
  if (F7)
    moving = __syncthreads_or(mv);
  else
    __syncthreads();

  // ---- P7: Lagrangian update of zones [3, zmax-1] -> PRIM ----------------
  if (live && s >= 3 && s <= zmax - 1) {
    const double dx0 = __ldg(A.dx + q);
    const double dxp = dx0 + dt * (CF[ci + SS] - CF[ci]);
    if (!(dxp > 0.0)) {
      atomicMin(s_err, err_key(*A.step, A.phase, AXIS,
                               (pencil_index() << 20) | ((unsigned long long)q << 2) |
                                   kErrStepRejected));
    } else {
      double u[8];
      Ops o;
      const double r_dxp = o.rcp(dxp);
      const double shrink = o.div(dx0, dxp, r_dxp);
#pragma unroll
      for (int v = 0; v < 8; ++v)
        u[v] = CONS[v * T + ci] * shrink -
               o.div(dt * (SA[v * T + ci + SS] - SA[v * T + ci]), dxp, r_dxp);
      const double internal =
          (u[kPE] - o.dv(0.5 * ((u[kUn] * u[kUn] + u[kUt1] * u[kUt1]) + u[kUt2] * u[kUt2]),
                         u[kRho])) -
          o.div((u[kBn] * u[kBn] + u[kBt1] * u[kBt1]) + u[kBt2] * u[kBt2], c.two_mu0,
                k.r_two_mu0);
      tbad |= o.bad;
#pragma unroll
      for (int v = 0; v < 8; ++v) PRIM[v * T + ci] = u[v];
      if (c.pressure_floor <= 0.0 && (!(u[kRho] > 0.0) || !(internal > 0.0)))
        atomicMin(s_err, err_key(*A.step, A.phase, AXIS,
                                 (pencil_index() << 20) | ((unsigned long long)q << 2) |
                                     kErrLagUnphysical));
    }
  }
  const bool e8 = live && s >= 4 && s <= TLv - 4;
  if (F7) {
    // ---- P7b in P7's phase: conserved slopes -> TR (dead since P3; CONS
    // is untouched by P7), only in tiles with a moving edge
    if (moving && live && s >= 1 && s <= TLv - 2) {
      const SlopeC sc = slope_coef(A.slope, q);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const double* cv = CONS + v * T + ci;
        TR[v * T + ci] = slope_with(cv[-SS], cv[0], cv[SS], sc);
      }
    }
    __syncthreads();
  } else {
#if PPMLR_SWEEP_CSLOPE
  // ---- P7b: conserved slopes at s in [1, TLv-2] -> SA (fluxes are dead) --
  // Only tiles with a moving edge remap anything; the decision is uniform
  // across the CTA, so the extra barrier is legal.
  if (__syncthreads_or(e8 && CF[ci] * dt != 0.0)) {
    if (live && s >= 1 && s <= TLv - 2) {
      const SlopeC sc = slope_coef(A.slope, q);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const double* cv = CONS + v * T + ci;
        SA[v * T + ci] = slope_with(cv[-SS], cv[0], cv[SS], sc);
      }
    }
    __syncthreads();
  }
#else
  __syncthreads();
#endif
  }

  // ---- P8: slivers at edges [4, TLv-4] (moving edges only) ---------------
  double sl[8];
  if (e8) {
    const double delta = CF[ci] * dt;
#pragma unroll
    for (int v = 0; v < 8; ++v) sl[v] = 0.0;
    if (delta != 0.0) {
      const bool right = delta > 0.0;
      const int kc = right ? ci - SS : ci;  // upwind zone
      const int kq = right ? q - 1 : q;
      const double width = __ldg(A.dx + kq) + dt * (CF[kc + SS] - CF[kc]);
      double e0[kQfcN], e1[kQfcN];
#if !PPMLR_SWEEP_CSLOPE
      SlopeC sc[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) sc[j] = slope_coef(A.slope, kq - 1 + j);
#endif
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
        const double* cv = CONS + v * T + kc;
        auto win = [&](int j) { return cv[j * SS]; };
        double al, ar, six;
#if PPMLR_SWEEP_CSLOPE
        const double* dv = (F7 ? TR : SA) + v * T + kc;
        auto dwin = [&](int j) { return dv[j * SS]; };
        zone_parabola_dm(win, dwin, e0, e1, k, o, al, ar, six);
#else
        zone_parabola(win, sc, e0, e1, k, o, al, ar, six);
#endif
        const double mean =
            right ? avg_right(al, ar, six, hs, tw) : avg_left(al, ar, six, hs, tw);
        sl[v] = delta * (mean + (PRIM[v * T + kc] - cv[0]));
      }
      tbad |= o.bad;
    }
  }
  if (F7) {  // SA (fluxes) is dead since P7: no write-after-read hazard
    if (e8) {
#pragma unroll
      for (int v = 0; v < 8; ++v) SA[v * T + ci] = sl[v];
    }
    __syncthreads();
  } else if (XS) {  // TR (left states) is dead since P4: no write-after-read hazard
    if (e8) {
#pragma unroll
      for (int v = 0; v < 8; ++v) TR[v * T + ci] = sl[v];
    }
    __syncthreads();
  } else {
    __syncthreads();
    if (e8) {
#pragma unroll
      for (int v = 0; v < 8; ++v) CONS[v * T + ci] = sl[v];
    }
    __syncthreads();
  }
  const double* SL = F7 ? SA : (XS ? TR : CONS);  // slivers
  double* OUT = F7 ? TR : SA;  // TMA store staging (dead slots)

  // ---- P9: remap, cons_to_prim, store (zones [4, TLv-5]) ----------------
  if (live && s >= 4 && s <= TLv - 5) {
    const double dxe = __ldg(A.dx + q);
    const double r_dxe = __ldg(A.rdx + q);
    const double width = dxe + dt * (CF[ci + SS] - CF[ci]);
    double out[8], u[8], cs[8];
    Ops o;
    const double scale = o.div(width, dxe, r_dxe);
#pragma unroll
    for (int v = 0; v < 8; ++v)
      u[v] = PRIM[v * T + ci] * scale + o.div(SL[v * T + ci] - SL[v * T + ci + SS], dxe, r_dxe);
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
    } else if (tma_store) {
      // dense box order of the L interior zones x NP pencils (OUT is dead)
      const int bi = AXIS == 0 ? p * A.L + (s - 4) : (s - 4) * NP + p;
#pragma unroll
      for (int f = 0; f < 8; ++f) OUT[f * T + bi] = out[f];
    } else {
      const long long off = base + (long long)p * A.stride_g + (long long)s * A.stride_a;
#pragma unroll
      for (int f = 0; f < 8; ++f) A.dst[f][off] = out[f];
    }
  }
  if (tma_store) {
    // whole tile: the caller sends the L x NP box of every field out with
    // TMA after its closing barrier (the stores' smem writes are made
    // visible to the async proxy here)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (store) {
      const int a0 = seg0 + 4, g = g0 + 4, o = oc + 4;
      store[0] = (int)(OUT - smem) / T;  // first slot of the staged box (may be 0)
      store[1] = AXIS == 0 ? a0 : g;
      store[2] = AXIS == 0 ? g : (AXIS == 1 ? a0 : o);
      store[3] = AXIS == 2 ? a0 : o;
    }
  }
  return tbad;
}

#ifdef PPMLR_FAST_MATH
using MainOps = FastMathOps;  // tolerance-gated fast mode
#else
using MainOps = FastOps;      // bit-exact replay of nvcc's fast paths
#endif


// Main instance: every tile with MainOps; a tile whose guards all held
// commits its error keys and results, otherwise it is queued for EXACT,
// which re-runs the queued tiles with plain `/` and `sqrt`.
template <int AXIS, bool DIPOLE, int NP, int TLC, bool EXACT>
__global__ void __launch_bounds__(NP * kSweepTL, PPMLR_SWEEP_MINB)
    sweep_kernel(const SweepArgs A, const __grid_constant__ SweepMaps M) {
  extern __shared__ __align__(128) double smem[];
  __shared__ unsigned long long s_err;
  __shared__ __align__(8) unsigned long long s_mbar;
  if (EXACT) {
    const unsigned n = *A.redo_count;
    for (unsigned i = blockIdx.x; i < n; i += gridDim.x) {
      if (threadIdx.x == 0) s_err = kNoError;
      __syncthreads();
      const TileId id = tile_of(A, (int)A.redo_list[i]);
      sweep_tile<AXIS, DIPOLE, NP, TLC, ExactOps>(A, id.seg, id.grp, id.oc, smem, &s_err);
      __syncthreads();
      if (threadIdx.x == 0 && s_err != kNoError) atomicMin(A.err, s_err);
      __syncthreads();
    }
    return;
  }
  // grid = (nseg, ngroups, no): the tile coordinates need no division.
  // The tile's inputs stream in with TMA (boxes sized to the block's tile).
  constexpr bool kTma = PPMLR_SWEEP_TMA;
  // the split coordinate (segment for x, pencil group for y/z) of a part launch
  const int seg = AXIS == 0 ? split_unit(A.part, A.cl, A.cr, blockIdx.x) : (int)blockIdx.x;
  const int grp = AXIS == 0 ? (int)blockIdx.y : split_unit(A.part, A.cl, A.cr, blockIdx.y);
  if (threadIdx.x == 0) {
    s_err = kNoError;
    if (kTma) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_mbar)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tma_load_tile<AXIS, DIPOLE, NP, TLC>(A, M, seg, grp, blockIdx.z, smem, &s_mbar);
    }
  }
  __syncthreads();
  // store[0]: first smem slot of the staged result box, -1 = no TMA store
  int store[4] = {-1, 0, 0, 0};
  const bool bad = sweep_tile<AXIS, DIPOLE, NP, TLC, MainOps, kTma>(
      A, seg, grp, blockIdx.z, smem, &s_err, &s_mbar, store);
  // one closing barrier: the tile's results are in shared memory and its
  // flags are final
  const bool any_bad = __syncthreads_or(bad);
  if (threadIdx.x == 0 && store[0] >= 0) {
    // a flagged tile is re-run and rewritten by the exact instance later in
    // stream order, so its box may go out regardless
#pragma unroll
    for (int f = 0; f < 8; ++f)
      asm volatile(
          "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
              reinterpret_cast<unsigned long long>(&M.out[f])),
          "r"(store[1]), "r"(store[2]), "r"(store[3]),
          "r"(smem_u32(smem + store[0] * slot_stride(NP * (TLC > 0 ? TLC : A.L + 8)) +
                       f * slot_stride(NP * (TLC > 0 ? TLC : A.L + 8))))
          : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  if (any_bad) {
    if (threadIdx.x == 0)
      A.redo_list[atomicAdd(A.redo_count, 1u)] =
          seg + A.nseg * (grp + A.ngroups * blockIdx.z);
  } else if (threadIdx.x == 0 && s_err != kNoError) {
    atomicMin(A.err, s_err);
  }
  // the shared memory must outlive the stores' reads of it
  if (threadIdx.x == 0 && store[0] >= 0)
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

}  // namespace PPMLR_KNS
}  // namespace ppmlr_b200
