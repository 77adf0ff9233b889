// Directional PPMLR sweep kernel (sm_100a, FP64): the whole of the
// reference's sweep_axis -> sweep_1d (proj/src/stepper.cpp:249-282,
// proj/src/ppm1d.cpp:111-364) for every pencil of one block along AXIS.
//
// Work decomposition.  A CTA owns a tile of NP adjacent pencils x one
// segment of TL = L + 8 strip positions (L interior cells plus the 4-cell
// dependency halo on each side).  The tile is staged in
// shared memory, structure-of-arrays, and the 1-D algorithm runs as a
// sequence of cell-parallel phases separated by __syncthreads():
//
//   P0 load + strip-frame prim/cons + c_f       P5 (fused in P4) cons slopes
//   P1 prim slopes           P2 prim interfaces P6 cons interfaces
//   P3 prim parabolas -> traced L/R states      P7 Lagrangian update + checks
//   P4 edge Riemann solve -> u*, fluxes         P8 remap slivers (once per edge)
//                                               P9 remap + cons_to_prim + store
//
// Shared-memory slots (T = NP*TL doubles each) are recycled across phases:
//   PRIM[8]  prim -> traced R -> cons interface values
//   CONS[8]  cons (live to the end)
//   CF       c_f -> u*
//   A[8]     prim slopes -> traced L -> cons slopes -> Lagrangian state
//   B[8]     prim interface values -> fluxes -> slivers
//   BD[3]    dipole field (DIPOLE only)
//
// Results are bit-identical to the reference in the strict build: each
// output is produced by the reference's own expression sequence; the only
// reorganisations are exact (hoisted geometry, sliver/sigma terms evaluated
// once per edge instead of twice, segment halos recomputed).
#pragma once
#include "ppmlr_dev.cuh"

namespace ppmlr_b200 {

// Compile-time tile length of the main sweep instantiation (L = 64 interior
// cells per segment, 4 pencils per tile).
constexpr int kSweepTL = 72;

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

// TLC > 0: compile-time tile length (TL = TLC = L + 8, constant smem strides);
// TLC == 0: runtime TL = A.L + 8.
// One tile of the sweep with arithmetic policy Ops.  Returns true when a
// FastOps guard failed somewhere in the tile (its results and error keys
// are then discarded and the tile is re-run with ExactOps).  Error keys go
// to *s_err (shared) and are committed by the caller.
template <int AXIS, bool DIPOLE, int NP, int TLC, class Ops>
__device__ __forceinline__ bool sweep_tile(const SweepArgs& A, const int bid, double* smem,
                                           unsigned long long* s_err) {
  bool tbad = false;
  const int TL = TLC > 0 ? TLC : A.L + 8;
  const int T = NP * TL;
  double* PRIM = smem;
  double* CONS = smem + 8 * T;
  double* CF = smem + 16 * T;
  double* SA = smem + 17 * T;
  double* SB = smem + 25 * T;
  double* BD = smem + 33 * T;
  // Neighbour offset along the strip inside the tile.
  const int SS = AXIS == 0 ? 1 : NP;

  const int seg = bid % A.nseg;
  const int rest = bid / A.nseg;
  const int grp = rest % A.ngroups;
  const int oc = rest / A.ngroups;
  const int nn = A.n + 8;
  const int seg0 = seg * A.L;
  const int TLv = min(TL, nn - seg0);
  const bool final_seg = seg == A.nseg - 1;
  const int zmax = final_seg ? TLv - 2 : TL - 3;  // last zone with traced states
  const int g0 = grp * NP;
  const int npv = min(NP, A.ng - g0);
  const double dt = *A.dt;
  const Consts& c = A.c;
  const KC k = make_kc(c);
  const long long base = (long long)(g0 + 4) * A.stride_g + (long long)(oc + 4) * A.stride_o +
                         (long long)seg0 * A.stride_a;

  auto decode = [&](int ci, int& s, int& p) {
    if (AXIS == 0) {
      p = ci / TL;
      s = ci - p * TL;
    } else {
      s = ci / NP;
      p = ci - s * NP;
    }
  };
  // Reference pencil index t1 + nb*t2 for tile pencil p (error ordering).
  auto pencil_index = [&](int p) -> unsigned long long {
    const int gcoord = g0 + p;
    int t1, t2;
    if (AXIS == 0) {  // b = y (group), d = z (other)
      t1 = gcoord;
      t2 = oc;
    } else if (AXIS == 1) {  // b = z (other), d = x (group)
      t1 = oc;
      t2 = gcoord;
    } else {  // b = x (group), d = y (other)
      t1 = gcoord;
      t2 = oc;
    }
    return (unsigned long long)t1 + (unsigned long long)A.nb * (unsigned long long)t2;
  };

  // ---- P0: load, strip-frame primitives, conserved, c_f ----------------
  for (int ci = threadIdx.x; ci < T; ci += blockDim.x) {
    int s, p;
    decode(ci, s, p);
    if (s >= TLv || p >= npv) continue;
    const long long off = base + (long long)p * A.stride_g + (long long)s * A.stride_a;
    double q[8];
#pragma unroll
    for (int f = 0; f < 8; ++f) q[f] = __ldg(A.src[f] + off);
    double b0 = 0.0, b1 = 0.0, b2 = 0.0;
    if (DIPOLE) {
      b0 = __ldg(A.bd[0] + off);
      b1 = __ldg(A.bd[1] + off);
      b2 = __ldg(A.bd[2] + off);
      // strip order (a, a+1, a+2)
      BD[0 * T + ci] = AXIS == 0 ? b0 : (AXIS == 1 ? b1 : b2);
      BD[1 * T + ci] = AXIS == 0 ? b1 : (AXIS == 1 ? b2 : b0);
      BD[2 * T + ci] = AXIS == 0 ? b2 : (AXIS == 1 ? b0 : b1);
    }
    constexpr int a = AXIS, b = (AXIS + 1) % 3, d = (AXIS + 2) % 3;
    double w[8];
    w[kRho] = q[0];
    w[kUn] = q[1 + a];
    w[kUt1] = q[1 + b];
    w[kUt2] = q[1 + d];
    w[kBn] = q[4 + a];
    w[kBt1] = q[4 + b];
    w[kBt2] = q[4 + d];
    w[kPE] = q[7];
    double cf = 0.0, e = 0.0;
    {
      Ops o;
      cf = fast_speed3<AXIS>(q, b0, b1, b2, k, o);
      e = strip_energy(w, k, o);
      tbad |= o.bad;
    }
    CF[ci] = cf;
#pragma unroll
    for (int v = 0; v < 8; ++v) PRIM[v * T + ci] = w[v];
    CONS[kRho * T + ci] = w[kRho];
    CONS[kUn * T + ci] = w[kRho] * w[kUn];
    CONS[kUt1 * T + ci] = w[kRho] * w[kUt1];
    CONS[kUt2 * T + ci] = w[kRho] * w[kUt2];
    CONS[kBn * T + ci] = w[kBn];
    CONS[kBt1 * T + ci] = w[kBt1];
    CONS[kBt2 * T + ci] = w[kBt2];
    CONS[kPE * T + ci] = e;
  }
  __syncthreads();

  // ---- P1: primitive slopes at s in [1, TLv-2] -------------------------
  for (int ci = threadIdx.x; ci < T; ci += blockDim.x) {
    int s, p;
    decode(ci, s, p);
    if (s < 1 || s > TLv - 2 || p >= npv) continue;
    const double* gc = A.slope + 3 * (seg0 + s);
    const double c0 = __ldg(gc), cA = __ldg(gc + 1), cB = __ldg(gc + 2);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const double* q = PRIM + v * T + ci;
      SA[v * T + ci] = limited_slope(q[-SS], q[0], q[SS], c0, cA, cB);
    }
  }
  __syncthreads();

  // ---- P2: primitive interface values at edges m in [2, TLv-2] ---------
  for (int ci = threadIdx.x; ci < T; ci += blockDim.x) {
    int s, p;
    decode(ci, s, p);
    if (s < 2 || s > TLv - 2 || p >= npv) continue;
    double e[5];
    const double* ge = A.qfc + 5 * (seg0 + s);
#pragma unroll
    for (int kk = 0; kk < 5; ++kk) e[kk] = __ldg(ge + kk);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const double* q = PRIM + v * T + ci;
      const double* dm = SA + v * T + ci;
      SB[v * T + ci] = interface_value(q[-SS], q[0], dm[-SS], dm[0], e);
    }
  }
  __syncthreads();

  // ---- P3: primitive parabolas -> traced edge states of zone s ---------
  for (int ci = threadIdx.x; ci < T; ci += blockDim.x) {
    int s, p;
    decode(ci, s, p);
    if (s < 2 || s > zmax || p >= npv) continue;
    const int q = seg0 + s;
    const bool flat = q < 2 || q >= nn - 2;
    const double dxq = __ldg(A.dx + q), rdxq = __ldg(A.rdx + q);
    double L[8], R[8];
    {
      Ops o;
      const double sigma = sclamp(o.div(CF[ci] * dt, dxq, rdxq), 0.0, 1.0);
      const double hs = 0.5 * sigma;
      const double tw = tw_of(sigma, k, o);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const double av = PRIM[v * T + ci];
        double al = flat ? av : SB[v * T + ci], ar = flat ? av : SB[v * T + ci + SS], six;
        limit_parabola(al, ar, av, six, k, o);
        L[v] = avg_left(al, ar, six, hs, tw);
        R[v] = avg_right(al, ar, six, hs, tw);
      }
      tbad |= o.bad;
    }
    const bool badL = !(L[kRho] > 0.0) || !(L[kPE] > 0.0);
    const bool badR = !(R[kRho] > 0.0) || !(R[kPE] > 0.0);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      if (!badL) SA[v * T + ci] = L[v];
      else SA[v * T + ci] = PRIM[v * T + ci];
      if (!badR) PRIM[v * T + ci] = R[v];
    }
  }
  __syncthreads();

  // ---- P4: edge solve at m in [3, zmax]; P5: cons slopes (same cell) ---
  for (int ci = threadIdx.x; ci < T; ci += blockDim.x) {
    int s, p;
    decode(ci, s, p);
    if (p >= npv) continue;
    if (s >= 3 && s <= zmax) {
      double f[8], bl[3] = {0.0, 0.0, 0.0}, br[3] = {0.0, 0.0, 0.0};
      const SmemVec ql{PRIM + ci - SS, T}, qr{SA + ci, T};
      if (DIPOLE) {
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
          bl[kk] = BD[kk * T + ci - SS];
          br[kk] = BD[kk * T + ci];
        }
      }
      double us = 0.0;
      {
      Ops o;
        us = solve_edge(ql, qr, bl, br, k, f, o);
        tbad |= o.bad;
      }
      CF[ci] = us;
#pragma unroll
      for (int v = 0; v < 8; ++v) SB[v * T + ci] = f[v];
    }
    if (s >= 1 && s <= TLv - 2) {
      const double* gc = A.slope + 3 * (seg0 + s);
      const double c0 = __ldg(gc), cA = __ldg(gc + 1), cB = __ldg(gc + 2);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const double* q = CONS + v * T + ci;
        SA[v * T + ci] = limited_slope(q[-SS], q[0], q[SS], c0, cA, cB);
      }
    }
  }
  __syncthreads();

  // ---- P6: conserved interface values at m in [2, TLv-2] -> PRIM slots ---
  for (int ci = threadIdx.x; ci < T; ci += blockDim.x) {
    int s, p;
    decode(ci, s, p);
    if (s < 2 || s > TLv - 2 || p >= npv) continue;
    double e[5];
    const double* ge = A.qfc + 5 * (seg0 + s);
#pragma unroll
    for (int kk = 0; kk < 5; ++kk) e[kk] = __ldg(ge + kk);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const double* q = CONS + v * T + ci;
      const double* dm = SA + v * T + ci;
      PRIM[v * T + ci] = interface_value(q[-SS], q[0], dm[-SS], dm[0], e);
    }
  }
  __syncthreads();

  // ---- P7: Lagrangian update of zones k in [3, zmax-1] + checks ----------
  for (int ci = threadIdx.x; ci < T; ci += blockDim.x) {
    int s, p;
    decode(ci, s, p);
    if (s < 3 || s > zmax - 1 || p >= npv) continue;
    const int q = seg0 + s;
    const double dx0 = __ldg(A.dx + q);
    const double dxp = dx0 + dt * (CF[ci + SS] - CF[ci]);
    if (!(dxp > 0.0)) {
      atomicMin(s_err, err_key(*A.step, A.phase, AXIS,
                               (pencil_index(p) << 20) | ((unsigned long long)q << 2) |
                                   kErrStepRejected));
      continue;
    }
    double u[8], internal = 0.0;
    {
      Ops o;
      const double r_dxp = o.rcp(dxp);
      const double shrink = o.div(dx0, dxp, r_dxp);
#pragma unroll
      for (int v = 0; v < 8; ++v)
        u[v] = CONS[v * T + ci] * shrink -
               o.div(dt * (SB[v * T + ci + SS] - SB[v * T + ci]), dxp, r_dxp);
      internal =
          (u[kPE] - o.dv(0.5 * ((u[kUn] * u[kUn] + u[kUt1] * u[kUt1]) + u[kUt2] * u[kUt2]),
                         u[kRho])) -
          o.div((u[kBn] * u[kBn] + u[kBt1] * u[kBt1]) + u[kBt2] * u[kBt2], c.two_mu0,
                k.r_two_mu0);
      tbad |= o.bad;
    }
#pragma unroll
    for (int v = 0; v < 8; ++v) SA[v * T + ci] = u[v];
    if (c.pressure_floor <= 0.0 && (!(u[kRho] > 0.0) || !(internal > 0.0)))
      atomicMin(s_err, err_key(*A.step, A.phase, AXIS,
                               (pencil_index(p) << 20) | ((unsigned long long)q << 2) |
                                   kErrLagUnphysical));
  }
  __syncthreads();

  // ---- P8: remap slivers at edges m in [4, TLv-4] -> SB ------------------
  for (int ci = threadIdx.x; ci < T; ci += blockDim.x) {
    int s, p;
    decode(ci, s, p);
    if (s < 4 || s > TLv - 4 || p >= npv) continue;
    const int m = seg0 + s;
    const double delta = CF[ci] * dt;
    double sl[8];
    if (delta == 0.0) {
#pragma unroll
      for (int v = 0; v < 8; ++v) sl[v] = 0.0;
    } else {
      // upwind zone k: m-1 (delta > 0, right part) or m (delta < 0, left part)
      const bool right = delta > 0.0;
      const int kc = right ? ci - SS : ci;
      const int kq = right ? m - 1 : m;
      const double width = __ldg(A.dx + kq) + dt * (CF[kc + SS] - CF[kc]);
      {
      Ops o;
        const double sigma = o.dv(right ? delta : -delta, width);
        const double hs = 0.5 * sigma;
        const double tw = tw_of(sigma, k, o);
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const double av = CONS[v * T + kc];
          double al = PRIM[v * T + kc], ar = PRIM[v * T + kc + SS], six;
          limit_parabola(al, ar, av, six, k, o);
          const double mean =
              right ? avg_right(al, ar, six, hs, tw) : avg_left(al, ar, six, hs, tw);
          sl[v] = delta * (mean + (SA[v * T + kc] - av));
        }
        tbad |= o.bad;
      }
    }
#pragma unroll
    for (int v = 0; v < 8; ++v) SB[v * T + ci] = sl[v];
  }
  __syncthreads();

  // ---- P9: remap onto the fixed mesh, cons_to_prim, store ---------------
  for (int ci = threadIdx.x; ci < T; ci += blockDim.x) {
    int s, p;
    decode(ci, s, p);
    if (s < 4 || s > TLv - 5 || p >= npv) continue;
    const int q = seg0 + s;
    const double dxe = __ldg(A.dx + q);
    const double r_dxe = __ldg(A.rdx + q);
    const double width = dxe + dt * (CF[ci + SS] - CF[ci]);
    double out[8];
    constexpr int a = AXIS, b = (AXIS + 1) % 3, d = (AXIS + 2) % 3;
    int bad = 0;
    {
      Ops o;
      const double scale = o.div(width, dxe, r_dxe);
      double u[8];
#pragma unroll
      for (int v = 0; v < 8; ++v)
        u[v] = SA[v * T + ci] * scale + o.div(SB[v * T + ci] - SB[v * T + ci + SS], dxe, r_dxe);
      double cs[8];
      cs[0] = u[kRho];
      cs[1 + a] = u[kUn];
      cs[1 + b] = u[kUt1];
      cs[1 + d] = u[kUt2];
      cs[4 + a] = u[kBn];
      cs[4 + b] = u[kBt1];
      cs[4 + d] = u[kBt2];
      cs[7] = u[kPE];
      bad = cons_to_prim3(cs, out, k, o);
      tbad |= o.bad;
    }
    if (bad) {
      atomicMin(s_err, err_key(*A.step, A.phase, AXIS,
                               (pencil_index(p) << 20) | (1ull << 19) |
                                   ((unsigned long long)(q - 4) << 2) |
                                   (bad == 1 ? kErrDensity : kErrPressure)));
      continue;
    }
    const long long off = base + (long long)p * A.stride_g + (long long)s * A.stride_a;
#pragma unroll
    for (int f = 0; f < 8; ++f) A.dst[f][off] = out[f];
  }
  return tbad;
}

#ifdef PPMLR_FAST_MATH
using MainOps = FastMathOps;  // tolerance-gated fast mode
#else
using MainOps = FastOps;      // bit-exact replay of nvcc's fast paths
#endif

// FAST instance: every tile with MainOps; a tile whose guards all held
// commits its error keys and results, otherwise it is queued for EXACT.
// EXACT instance: re-runs the queued tiles with plain `/` and `sqrt`.
template <int AXIS, bool DIPOLE, int NP, int TLC, bool EXACT>
__global__ void __launch_bounds__(TLC > 0 ? NP * TLC : 512, TLC > 0 ? 2 : 1)
    sweep_kernel(const SweepArgs A) {
  extern __shared__ double smem[];
  __shared__ unsigned long long s_err;
  if (EXACT) {
    const unsigned n = *A.redo_count;
    for (unsigned i = blockIdx.x; i < n; i += gridDim.x) {
      if (threadIdx.x == 0) s_err = kNoError;
      __syncthreads();
      sweep_tile<AXIS, DIPOLE, NP, TLC, ExactOps>(A, (int)A.redo_list[i], smem, &s_err);
      __syncthreads();
      if (threadIdx.x == 0 && s_err != kNoError) atomicMin(A.err, s_err);
      __syncthreads();
    }
    return;
  }
  if (threadIdx.x == 0) s_err = kNoError;
  __syncthreads();
  const bool bad = sweep_tile<AXIS, DIPOLE, NP, TLC, MainOps>(A, blockIdx.x, smem, &s_err);
  if (__syncthreads_or(bad)) {
    if (threadIdx.x == 0) A.redo_list[atomicAdd(A.redo_count, 1u)] = blockIdx.x;
  } else if (threadIdx.x == 0 && s_err != kNoError) {
    atomicMin(A.err, s_err);
  }
}


}  // namespace PPMLR_KNS
}  // namespace ppmlr_b200
