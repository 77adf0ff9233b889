// Host-side planning code and the in-process Harness over device blocks.
//
// Native C++ restatement (not a copy) of the reference's host layer that
// feeds the hot path: stretched-axis construction (proj/src/grid.cpp),
// partition validation/layout (proj/src/decomp.cpp), ghost-extended block
// geometry and the dipole field (proj/src/stepper.cpp:17-71,
// proj/src/physics.cpp:14-27), the initial conditions, and Harness::advance
// (proj/src/harness.cpp) driving device blocks.  Compiled with
// -ffp-contract=off so every geometry value is bit-identical to the
// reference's (they feed the bit-exact strict kernels).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <thread>
#include <string>
#include <vector>

#include "block.hpp"

using namespace ppmlr_b200;

namespace {

constexpr double kPi = 3.14159265358979323846;

struct SpecError : std::runtime_error {
  int code;
  SpecError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void invalid(const std::string& m) { throw SpecError(PPMLR_INVALID_SPEC, m); }

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const SpecError& e) {
    set_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return PPMLR_RUNTIME;
  }
}

// ------------------------------------------------------------- axis build

struct Axis {
  std::vector<double> edges, centers, spacings;
  int n() const { return (int)spacings.size(); }
};

// grid.cpp:9-17 semantics: sum d*r^1..d*r^n term by term.
double geometric_sum(double d, double r, int n) {
  double term = d, sum = 0.0;
  for (int k = 0; k < n; ++k) {
    term *= r;
    sum += term;
  }
  return sum;
}

double closing_ratio(double d, double extent, int n, const char* side) {
  const double at_one = d * n;
  const double tol = 1e-12 * std::max(1.0, extent);
  if (std::abs(at_one - extent) <= tol) return 1.0;
  if (at_one > extent)
    invalid(std::string("axis ") + side +
            " side: allocated cells overfill the side at ratio 1 (no closing ratio >= 1 exists)");
  if (geometric_sum(d, 2.0, n) < extent)
    invalid(std::string("axis ") + side +
            " side: no ratio in (1, 2] closes the side for the allocated cell count");
  double lo = 1.0, hi = 2.0;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid == lo || mid == hi) break;
    if (geometric_sum(d, mid, n) < extent)
      lo = mid;
    else
      hi = mid;
  }
  return 0.5 * (lo + hi);
}

Axis make_axis(const ppmlr_axis_spec& s) {
  if (!(s.d_uniform > 0.0)) invalid("d_uniform must be positive");
  if (!(s.ratio > 1.0)) invalid("nominal_ratio must exceed 1");
  if (!(s.min <= s.uniform_lo && s.uniform_lo < s.uniform_hi && s.uniform_hi <= s.max))
    invalid("axis spec requires min <= uniform_lo < uniform_hi <= max");
  const double m = (s.uniform_hi - s.uniform_lo) / s.d_uniform;
  const double rounded = std::round(m);
  if (std::abs(m - rounded) > 1e-9 * std::max(1.0, m))
    invalid("uniform region extent is not an integer multiple of d_uniform");
  const int n_uniform = (int)rounded;
  const int n_stretch = s.cells - n_uniform;
  if (n_stretch < 0) invalid("target_cells smaller than the uniform cell count");
  const double len_lo = s.uniform_lo - s.min, len_hi = s.max - s.uniform_hi;
  if (len_lo == 0.0 && len_hi == 0.0 && n_stretch != 0)
    invalid("all-uniform axis but target_cells exceeds the uniform count");
  auto weight = [&](double len) {
    if (len <= 0.0) return 0.0;
    return std::log(1.0 + len * (s.ratio - 1.0) / s.d_uniform) / std::log(s.ratio);
  };
  int n_lo = 0, n_hi = 0;
  if (len_lo > 0.0 && len_hi > 0.0) {
    const double w_lo = weight(len_lo), w_hi = weight(len_hi);
    n_lo = (int)std::round(n_stretch * w_lo / (w_lo + w_hi));
    n_hi = n_stretch - n_lo;
  } else if (len_lo > 0.0) {
    n_lo = n_stretch;
  } else if (len_hi > 0.0) {
    n_hi = n_stretch;
  }
  if ((len_lo > 0.0 && n_lo <= 0) || (len_hi > 0.0 && n_hi <= 0))
    invalid("a stretched side received no cells; increase target_cells");
  const double r_lo = n_lo > 0 ? closing_ratio(s.d_uniform, len_lo, n_lo, "lower") : 1.0;
  const double r_hi = n_hi > 0 ? closing_ratio(s.d_uniform, len_hi, n_hi, "upper") : 1.0;
  const double cap = s.ratio + 0.05;
  if (r_lo > cap)
    invalid("lower side ratio " + std::to_string(r_lo) + " exceeds nominal_ratio + 0.05");
  if (r_hi > cap)
    invalid("upper side ratio " + std::to_string(r_hi) + " exceeds nominal_ratio + 0.05");
  const int n = n_lo + n_uniform + n_hi;
  Axis a;
  a.edges.assign(n + 1, 0.0);
  for (int k = 0; k <= n_uniform; ++k) a.edges[n_lo + k] = s.uniform_lo + k * s.d_uniform;
  double w = s.d_uniform;
  for (int k = 1; k <= n_lo; ++k) {
    w *= r_lo;
    a.edges[n_lo - k] = a.edges[n_lo - k + 1] - w;
  }
  w = s.d_uniform;
  for (int k = 1; k <= n_hi; ++k) {
    w *= r_hi;
    a.edges[n_lo + n_uniform + k] = a.edges[n_lo + n_uniform + k - 1] + w;
  }
  a.edges.front() = s.min;
  a.edges.back() = s.max;
  a.centers.resize(n);
  a.spacings.resize(n);
  for (int i = 0; i < n; ++i) {
    a.spacings[i] = a.edges[i + 1] - a.edges[i];
    a.centers[i] = 0.5 * (a.edges[i] + a.edges[i + 1]);
    if (!(a.spacings[i] > 0.0)) invalid("non-positive spacing at cell " + std::to_string(i));
  }
  return a;
}

// grid.cpp:137-145
int locate_cell(const Axis& a, double q) {
  if (q < a.edges.front() || q > a.edges.back())
    throw SpecError(PPMLR_OUT_OF_RANGE, "coordinate " + std::to_string(q) + " outside [" +
                                            std::to_string(a.edges.front()) + ", " +
                                            std::to_string(a.edges.back()) + "]");
  const auto it = std::lower_bound(a.edges.begin(), a.edges.end(), q);
  const int i = (int)(it - a.edges.begin());
  return std::clamp(i - 1, 0, a.n() - 1);
}

// ----------------------------------------------------------- decomposition

struct BlockPlan {
  int rank;
  int coords[3], lo[3], n[3], neighbor[6];
};

std::vector<std::string> violations_of(const int cnt[3], const Axis* ax) {
  std::vector<std::string> v;
  if (cnt[0] < 1 || cnt[1] < 1 || cnt[2] < 1) v.push_back("rank counts must be positive");
  if (cnt[1] % 2 == 0)
    v.push_back("ny = " + std::to_string(cnt[1]) + " is even; y and z rank counts must be odd");
  if (cnt[2] % 2 == 0)
    v.push_back("nz = " + std::to_string(cnt[2]) + " is even; y and z rank counts must be odd");
  const char name[3] = {'x', 'y', 'z'};
  for (int a = 0; a < 3; ++a) {
    const int r = cnt[a];
    if (r >= 1 && ax[a].n() % r != 0)
      v.push_back(std::string(1, name[a]) + " ranks " + std::to_string(r) + " do not divide " +
                  std::to_string(ax[a].n()) + " cells");
  }
  for (int a = 1; a < 3; ++a) {
    const int r = cnt[a];
    if (r < 1 || cnt[1] % 2 == 0 || cnt[2] % 2 == 0 || ax[a].n() % r != 0) continue;
    if (ax[a].edges.front() > 0.0 || ax[a].edges.back() < 0.0) continue;
    const int origin = locate_cell(ax[a], 0.0);
    if (origin / (ax[a].n() / r) != (r - 1) / 2)
      v.push_back(std::string("Earth-origin cell falls outside the middle ") + name[a] +
                  " block");
  }
  return v;
}

std::vector<BlockPlan> plan_layout(const int cnt[3], const Axis* ax, int* iono) {
  const auto v = violations_of(cnt, ax);
  if (!v.empty()) {
    std::string msg = "invalid partition:";
    for (const auto& s : v) msg += " [" + s + "]";
    invalid(msg);
  }
  int bc[3];
  for (int a = 0; a < 3; ++a) bc[a] = ax[a].n() / cnt[a];
  auto rank_of = [&](int x, int y, int z) { return x + cnt[0] * (y + cnt[1] * z); };
  std::vector<BlockPlan> out;
  for (int cz = 0; cz < cnt[2]; ++cz)
    for (int cy = 0; cy < cnt[1]; ++cy)
      for (int cx = 0; cx < cnt[0]; ++cx) {
        BlockPlan b;
        b.rank = rank_of(cx, cy, cz);
        const int c3[3] = {cx, cy, cz};
        for (int a = 0; a < 3; ++a) {
          b.coords[a] = c3[a];
          b.lo[a] = c3[a] * bc[a];
          b.n[a] = bc[a];
        }
        for (int a = 0; a < 3; ++a) {
          int lo[3] = {cx, cy, cz}, hi[3] = {cx, cy, cz};
          lo[a] -= 1;
          hi[a] += 1;
          b.neighbor[2 * a] = lo[a] >= 0 ? rank_of(lo[0], lo[1], lo[2]) : -1;
          b.neighbor[2 * a + 1] = hi[a] < cnt[a] ? rank_of(hi[0], hi[1], hi[2]) : -1;
        }
        out.push_back(b);
      }
  *iono = cnt[0] * cnt[1] * cnt[2];
  return out;
}

// stepper.cpp:17-39 ghost-extended local axis.
void local_axis(const Axis& ax, int lo, int n, int g, std::vector<double>& ce,
                std::vector<double>& sp) {
  const int span = n + 2 * g;
  ce.assign(span, 0.0);
  sp.assign(span, 0.0);
  for (int i = 0; i < span; ++i) {
    const int gi = lo + i - g;
    if (gi >= 0 && gi < ax.n()) {
      ce[i] = ax.centers[gi];
      sp[i] = ax.spacings[gi];
    }
  }
  for (int i = g - 1; i >= 0; --i) {
    if (lo + i - g >= 0) continue;
    sp[i] = sp[i + 1];
    ce[i] = ce[i + 1] - 0.5 * (sp[i] + sp[i + 1]);
  }
  for (int i = span - g; i < span; ++i) {
    if (lo + i - g < ax.n()) continue;
    sp[i] = sp[i - 1];
    ce[i] = ce[i - 1] + 0.5 * (sp[i] + sp[i - 1]);
  }
}

// ------------------------------------------------------------ physics init

struct V3 {
  double x, y, z;
};
inline double dot3(const V3& a, const V3& b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }

// physics.cpp:14-21 point dipole, moment m.
V3 dipole(const V3& pos, const V3& m, double mu0) {
  const double r2 = dot3(pos, pos);
  if (r2 == 0.0) throw SpecError(PPMLR_UNPHYSICAL, "dipole_field evaluated at the singularity");
  const double r = std::sqrt(r2);
  const V3 rh{pos.x / r, pos.y / r, pos.z / r};
  const double k = mu0 / (4.0 * kPi);
  const double s = 3.0 * dot3(m, rh);
  const V3 v{rh.x * s - m.x, rh.y * s - m.y, rh.z * s - m.z};
  const double den = r2 * r;
  return {(v.x * k) / den, (v.y * k) / den, (v.z * k) / den};
}

const V3 kMoment{0.0, 0.0, -4.0 * kPi};  // Constants::dipole_moment (physics.hpp:12)

struct Prim {
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};

// Synthetic ICs; must equal oracle/ref_shim.cpp make_ic (pinned by tests/golden).
std::function<Prim(const V3&)> make_ic(int kind, const double* p) {
  switch (kind) {
    case 0: {
      Prim u;
      for (int f = 0; f < 8; ++f) u.s[f] = p[f];
      return [u](const V3&) { return u; };
    }
    case 1:
      return [](const V3& r) {
        Prim q;
        const bool left = r.x < 0.5;
        q.s[0] = left ? 1.0 : 0.125;
        q.s[7] = left ? 1.0 : 0.1;
        q.s[4] = 0.75;
        q.s[5] = left ? 1.0 : -1.0;
        q.s[6] = 0.0;
        return q;
      };
    case 2: {
      const double g = p[0];
      return [g](const V3& r) {
        Prim q;
        q.s[0] = g * g;
        q.s[7] = g;
        q.s[1] = -std::sin(r.y);
        q.s[2] = std::sin(r.x);
        q.s[3] = 0.0;
        q.s[4] = -std::sin(r.y);
        q.s[5] = std::sin(2.0 * r.x);
        q.s[6] = 0.0;
        return q;
      };
    }
    case 3: {
      const double p_in = p[0], p_out = p[1], rad = p[2];
      return [=](const V3& r) {
        Prim q;
        const double cx = std::floor(r.x + 0.5);
        const double dx = r.x - cx;
        const double r2 = (dx * dx + r.y * r.y) + r.z * r.z;
        q.s[0] = 1.0;
        q.s[7] = r2 < rad * rad ? p_in : p_out;
        q.s[4] = std::sqrt(0.5);
        q.s[5] = std::sqrt(0.5);
        return q;
      };
    }
    case 4:
      return [](const V3& r) {
        const double w = std::exp(-dot3(r, r) / 2.0);
        Prim q;
        const double sv = 0.2 * w;
        q.s[0] = 1.0 + 0.3 * w;
        q.s[1] = (-r.y) * sv;
        q.s[2] = r.x * sv;
        q.s[3] = 0.0 * sv;
        q.s[4] = (-r.y) * 0.1;
        q.s[5] = r.x * 0.1;
        q.s[6] = 0.1 * 0.1;
        q.s[7] = 1.0 + 0.2 * w;
        return q;
      };
    case 5:
      return [](const V3& r) {
        const double w = std::exp(-0.5 * dot3(r, r));
        Prim q;
        q.s[0] = 1.0 + 0.3 * w;
        q.s[1] = 0.2 * w * -r.y;
        q.s[2] = 0.2 * w * r.x;
        q.s[3] = 0.0;
        q.s[4] = 0.1 * -r.y;
        q.s[5] = 0.1 * r.x;
        q.s[6] = 0.01;
        q.s[7] = 1.0 + 0.2 * w;
        return q;
      };
    case 6:
      return [](const V3& r) {
        Prim q;
        q.s[0] = 1.0;
        q.s[7] = 0.1 + 5.0 * std::exp(-dot3(r, r) / (0.25 * 0.25));
        return q;
      };
    default:
      invalid("unknown initial-condition kind " + std::to_string(kind));
  }
}

std::function<Prim(const V3&)> ic_of(int kind, const double* params) {
  double p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (params) std::memcpy(p, params, sizeof p);
  return make_ic(kind, p);
}

struct HostBlock {
  int n[3], lo[3], g;
  std::vector<double> cen[3], spc[3];
  V3 center(int i, int j, int k) const { return {cen[0][i], cen[1][j], cen[2][k]}; }
  size_t cells() const {
    return (size_t)(n[0] + 2 * g) * (n[1] + 2 * g) * (n[2] + 2 * g);
  }
};

// make_block's dipole (stepper.cpp:63-69) at one ghost-inclusive cell.
inline void dipole_cell(const HostBlock& hb, double mu0, int i, int j, int k, double* o) {
  const V3 v = dipole(hb.center(i, j, k), kMoment, mu0);
  o[0] = v.x;
  o[1] = v.y;
  o[2] = v.z;
}

struct MagnetosphereProfile {
  double rho_core, p_core, falloff, r_ref;
};

// init_magnetosphere (stepper.cpp:83-112) at one ghost-inclusive cell;
// `bd` is that cell's dipole (null without it).  Returns whether the cell
// belongs to the frozen inner core (interior and r < 3).
inline bool magnetosphere_cell(const HostBlock& hb, const ppmlr_gpu_options& o,
                               const MagnetosphereProfile& mp, const double* bd, int i, int j,
                               int k, double* s) {
  const int g = hb.g;
  const int S0 = hb.n[0] + 2 * g, S1 = hb.n[1] + 2 * g, S2 = hb.n[2] + 2 * g;
  const V3 image_m{-kMoment.x, kMoment.y, kMoment.z};
  const V3 pos = hb.center(i, j, k);
  for (int q = 0; q < 8; ++q) s[q] = 0.0;
  if (pos.x <= 15.0) {
    const double nrm = std::sqrt(dot3(pos, pos));
    const double rr = std::max(nrm, 1e-6);
    const double shape = std::pow(mp.r_ref / std::max(rr, mp.r_ref), mp.falloff);
    s[0] = mp.rho_core * shape;
    s[7] = mp.p_core * shape;
    const V3 b = dipole({pos.x - 30.0, pos.y - 0.0, pos.z - 0.0}, image_m, o.mu0);
    s[4] = b.x;
    s[5] = b.y;
    s[6] = b.z;
  } else {
    s[0] = o.wind_rho;
    s[7] = o.wind_p;
    for (int a = 0; a < 3; ++a) {
      s[1 + a] = o.wind_v[a];
      s[4 + a] = o.wind_imf[a] - (bd ? bd[a] : 0.0);
    }
  }
  const bool interior = i >= g && i < S0 - g && j >= g && j < S1 - g && k >= g && k < S2 - g;
  return interior && std::sqrt(dot3(pos, pos)) < 3.0;
}

// Runs fn(k, j, row_index) over the ghost-inclusive rows of k-planes
// [k0, k0 + nk) on worker threads; each worker owns a contiguous run of
// rows, so per-worker outputs concatenate back in (k, j, i) order.
void for_rows(const HostBlock& hb, int k0, int nk,
              const std::function<void(int w, int k, int j)>& fn, int nworkers) {
  const int S1 = hb.n[1] + 2 * hb.g;
  const long rows = (long)nk * S1;
  auto work = [&](int w) {
    const long r0 = rows * w / nworkers, r1 = rows * (w + 1) / nworkers;
    for (long r = r0; r < r1; ++r) fn(w, k0 + (int)(r / S1), (int)(r % S1));
  };
  if (nworkers == 1) {
    work(0);
    return;
  }
  std::vector<std::thread> pool;
  for (int w = 1; w < nworkers; ++w) pool.emplace_back(work, w);
  work(0);
  for (auto& t : pool) t.join();
}

int init_workers() {
  const unsigned hw = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(hw == 0 ? 1u : hw, 32u));
}

// Fills one k-chunk of the reference AoS layout (8 doubles per cell, plus
// the dipole when `bd` is non-null).  kind < 0: init_magnetosphere (frozen
// cells appended in (k, j, i) order); kind == -2: make_block's default
// {1, 0, 0, 1}; kind >= 0: init_with(make_ic(kind)).
struct ChunkInit {
  const HostBlock* hb;
  const ppmlr_gpu_options* o;
  int kind;
  MagnetosphereProfile mp{};
  std::function<Prim(const V3&)> ic;
  std::vector<int64_t>* fidx = nullptr;
  std::vector<double>* fst = nullptr;

  void operator()(int kr0, int nk, double* f, double* bd) const {
    const HostBlock& b = *hb;
    const int S0 = b.n[0] + 2 * b.g, S1 = b.n[1] + 2 * b.g;
    const int nw = (int)std::max(1L, std::min<long>(init_workers(), (long)nk * S1 / 4));
    std::vector<std::vector<int64_t>> wi(nw);
    std::vector<std::vector<double>> ws(nw);
    const bool need_bd = o->with_dipole && (bd || kind == -1);
    for_rows(b, kr0, nk, [&](int w, int k, int j) {
      double dloc[3];
      for (int i = 0; i < S0; ++i) {
        const size_t loc = (size_t)i + (size_t)S0 * (j + (size_t)S1 * (k - kr0));
        double* bc = nullptr;
        if (need_bd) {
          bc = bd ? bd + 3 * loc : dloc;
          dipole_cell(b, o->mu0, i, j, k, bc);
        }
        double* s = f + 8 * loc;
        if (kind == -1) {
          if (magnetosphere_cell(b, *o, mp, bc, i, j, k, s)) {
            wi[w].push_back((int64_t)i + (int64_t)S0 * (j + (int64_t)S1 * k));
            ws[w].insert(ws[w].end(), s, s + 8);
          }
        } else if (kind == -2) {
          for (int q = 0; q < 8; ++q) s[q] = 0.0;
          s[0] = 1.0;
          s[7] = 1.0;
        } else {
          const Prim p = ic(b.center(i, j, k));
          std::memcpy(s, p.s, 64);
        }
      }
    }, nw);
    if (fidx)
      for (int w = 0; w < nw; ++w) {
        fidx->insert(fidx->end(), wi[w].begin(), wi[w].end());
        fst->insert(fst->end(), ws[w].begin(), ws[w].end());
      }
  }
};

// Whole-block versions (ppmlr_host_block_state, block geometry queries).
void block_dipole(const HostBlock& hb, double mu0, std::vector<double>& bd) {
  const int S0 = hb.n[0] + 2 * hb.g, S1 = hb.n[1] + 2 * hb.g, S2 = hb.n[2] + 2 * hb.g;
  bd.assign((size_t)S0 * S1 * S2 * 3, 0.0);
  for (int k = 0; k < S2; ++k)
    for (int j = 0; j < S1; ++j)
      for (int i = 0; i < S0; ++i)
        dipole_cell(hb, mu0, i, j, k, &bd[3 * ((size_t)i + (size_t)S0 * (j + (size_t)S1 * k))]);
}

void block_fill(const HostBlock& hb, const ChunkInit& ci, std::vector<double>& f,
                std::vector<double>* bd) {
  const int S2 = hb.n[2] + 2 * hb.g;
  f.assign(hb.cells() * 8, 0.0);
  if (bd) bd->assign(hb.cells() * 3, 0.0);
  ci(0, S2, f.data(), bd ? bd->data() : nullptr);
}

HostBlock host_block(const Axis* ax, const BlockPlan& p, int g) {
  HostBlock hb;
  hb.g = g;
  for (int a = 0; a < 3; ++a) {
    hb.n[a] = p.n[a];
    hb.lo[a] = p.lo[a];
    local_axis(ax[a], p.lo[a], p.n[a], g, hb.cen[a], hb.spc[a]);
  }
  return hb;
}

}  // namespace

// ------------------------------------------------------------- harness

struct LedgerRow {  // LedgerEntry (exchange.hpp:40-46)
  long step;
  int transport;  // 0 staged, 1 direct
  long messages;
  uint64_t bytes;
  long copy_events;
};

struct ppmlr_gpu_harness {
  Axis ax[3];
  int cnt[3] = {1, 1, 1};
  std::vector<BlockPlan> plan;
  int iono = 0;
  ppmlr_gpu_options o{};
  std::vector<ppmlr_gpu_block*> blocks;
  std::vector<std::vector<double>> cen[3], spc[3];  // per block, ghost-inclusive (g_ref)
  std::vector<std::vector<int64_t>> fidx;
  std::vector<std::vector<double>> fst;
  long step = 0;
  double time = 0.0;
  // Multi-block layouts: one stream per block (on the block's device),
  // ordered with events (no host synchronisation inside a step); the global
  // dt is reduced on block 0's stream over the blocks' device slots.
  std::vector<int> devices;             // device of each block
  std::vector<cudaEvent_t> ev_state;    // block r's current state is complete
  cudaEvent_t ev_dt = nullptr;          // global dt written to every slot
  double** d_slots = nullptr;           // (block 0's device) each block's dt slot
  uint64_t ledger_bytes = 0;
  long ledger_messages = 0, ledger_events = 0;
  std::vector<LedgerRow> ledger;
  std::thread snap_writer;  // drains the last snapshot capture to its file
  int snap_rc = 0;
  std::string snap_err;

  int g() const { return o.ghost; }
  size_t cells(int r) const {
    const BlockPlan& p = plan[r];
    return (size_t)(p.n[0] + 2 * g()) * (p.n[1] + 2 * g()) * (p.n[2] + 2 * g());
  }
  V3 center(int r, int i, int j, int k) const {  // ghost-inclusive local indices
    return {cen[0][r][i], cen[1][r][j], cen[2][r][k]};
  }
};

namespace {

// Streams block r's initial state to the device chunk by chunk (the host
// never holds the whole block); the frozen core is collected on the way.
void upload_init(ppmlr_gpu_harness* h, int r, ChunkInit ci, bool with_bd) {
  const HostBlock hb = host_block(h->ax, h->plan[r], h->g());
  ci.hb = &hb;
  ci.o = &h->o;
  h->fidx[r].clear();
  h->fst[r].clear();
  if (ci.kind == -1) {
    ci.fidx = &h->fidx[r];
    ci.fst = &h->fst[r];
  }
  ppmlr_gpu_block* b = h->blocks[r];
  if (int e = block_upload_streamed(b, ci, with_bd)) throw SpecError(e, ppmlr_gpu_last_error());
  const auto& fi = h->fidx[r];
  if (int e = block_set_frozen(b, fi.empty() ? nullptr : fi.data(),
                               fi.empty() ? nullptr : h->fst[r].data(), (int64_t)fi.size()))
    throw SpecError(e, ppmlr_gpu_last_error());
}

// Device-side setup (block.cu block_init_device) for make_block's default
// state + dipole and init_with kinds 0..3; bit-identical to upload_init's
// host evaluation (tests/test_gpu_setup.py).  PPMLR_HOST_INIT=1 forces the
// host path.
bool use_device_init(int kind) {
  const char* e = std::getenv("PPMLR_HOST_INIT");
  return device_init_supported(kind) && !(e && std::atoi(e) != 0);
}

void init_device(ppmlr_gpu_harness* h, int r, int kind, const double* params, bool with_bd) {
  h->fidx[r].clear();
  h->fst[r].clear();
  ppmlr_gpu_block* b = h->blocks[r];
  if (int e = block_set_frozen(b, nullptr, nullptr, 0)) throw SpecError(e, ppmlr_gpu_last_error());
  double p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (params) std::memcpy(p, params, sizeof p);
  if (int e = block_init_device(b, kind, p, with_bd)) throw SpecError(e, ppmlr_gpu_last_error());
}

// Ledger entry of one exchange_step (exchange.cpp:93-149): every interior
// face both ways, payload face_cells*ghost*8 doubles; staged adds 6 copies.
void record_exchange(ppmlr_gpu_harness* h, long step) {
  LedgerRow e{step, h->o.transport, 0, 0, 0};
  for (const BlockPlan& b : h->plan)
    for (int face = 0; face < 6; ++face) {
      if (b.neighbor[face] < 0) continue;
      const int a = face / 2;
      const uint64_t payload =
          (uint64_t)b.n[(a + 1) % 3] * b.n[(a + 2) % 3] * h->g() * 8 * sizeof(double);
      e.messages += 1;
      e.bytes += payload;
      e.copy_events += 1 + (h->o.transport == 0 ? 6 : 0);
    }
  h->ledger.push_back(e);
  h->ledger_messages += e.messages;
  h->ledger_bytes += e.bytes;
  h->ledger_events += e.copy_events;
}

// ---------------------------------------------------------------- multi-block
// The reference Harness owns every block in one process (harness.hpp:79,
// harness.cpp:18-28).  Here each block lives on its own device (or several
// on one), issues on its own stream, and the blocks are ordered by CUDA
// events only: a halo copy on block r waits for its neighbour's state event,
// the global dt is a reduction over the blocks' device slots on block 0's
// stream.  The host synchronises once per advance()/run() window, to read
// the dt and the blocks' first-failure keys.

void multi_setup(ppmlr_gpu_harness* h) {
  const size_t nb = h->blocks.size();
  // peer access between every pair of devices in use (halo copies and the
  // dt reduction load and store across NVLink)
  std::vector<int> devs = h->devices;
  std::sort(devs.begin(), devs.end());
  devs.erase(std::unique(devs.begin(), devs.end()), devs.end());
  for (int a : devs)
    for (int b : devs) {
      if (a == b) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, a, b);
      if (!can)
        throw SpecError(PPMLR_RUNTIME, "no peer access from device " + std::to_string(a) +
                                           " to device " + std::to_string(b));
      cudaSetDevice(a);
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        throw SpecError(PPMLR_RUNTIME, std::string("cudaDeviceEnablePeerAccess: ") +
                                           cudaGetErrorString(e));
      cudaGetLastError();
    }
  h->ev_state.resize(nb);
  for (size_t r = 0; r < nb; ++r) {
    cudaSetDevice(h->devices[r]);
    if (cudaEventCreateWithFlags(&h->ev_state[r], cudaEventDisableTiming) != cudaSuccess)
      throw SpecError(PPMLR_RUNTIME, "cudaEventCreate failed");
  }
  cudaSetDevice(h->devices[0]);
  if (cudaEventCreateWithFlags(&h->ev_dt, cudaEventDisableTiming) != cudaSuccess ||
      cudaMalloc(&h->d_slots, sizeof(double*) * nb) != cudaSuccess)
    throw SpecError(PPMLR_RUNTIME, "multi-block setup: allocation failed");
  std::vector<double*> slots(nb);
  for (size_t r = 0; r < nb; ++r) slots[r] = ppmlr_gpu_block_dt_slot(h->blocks[r]);
  if (cudaMemcpy(h->d_slots, slots.data(), sizeof(double*) * nb, cudaMemcpyHostToDevice) !=
      cudaSuccess)
    throw SpecError(PPMLR_RUNTIME, "multi-block setup: slot table upload failed");
}

cudaStream_t stream_of(ppmlr_gpu_harness* h, size_t r) {
  return static_cast<cudaStream_t>(ppmlr_gpu_block_stream(h->blocks[r]));
}

#define MK(x)                                                                   \
  do {                                                                          \
    const cudaError_t e_ = (x);                                                 \
    if (e_ != cudaSuccess) throw SpecError(PPMLR_RUNTIME, cudaGetErrorString(e_)); \
  } while (0)

void record_states(ppmlr_gpu_harness* h) {
  for (size_t r = 0; r < h->blocks.size(); ++r) {
    MK(cudaSetDevice(h->devices[r]));
    MK(cudaEventRecord(h->ev_state[r], stream_of(h, r)));
  }
}

// compute_global_dt (harness.cpp:45-50): every slot holds cfl * local min
void multi_global_dt(ppmlr_gpu_harness* h) {
  record_states(h);
  cudaStream_t s0 = stream_of(h, 0);
  MK(cudaSetDevice(h->devices[0]));
  for (size_t r = 1; r < h->blocks.size(); ++r) MK(cudaStreamWaitEvent(s0, h->ev_state[r], 0));
  if (int e = launch_dt_min_all(h->d_slots, (int)h->blocks.size(), s0))
    throw SpecError(e, ppmlr_gpu_last_error());
  MK(cudaEventRecord(h->ev_dt, s0));
  for (size_t r = 1; r < h->blocks.size(); ++r) {
    MK(cudaSetDevice(h->devices[r]));
    MK(cudaStreamWaitEvent(stream_of(h, r), h->ev_dt, 0));
  }
}

// exchange_step + apply_boundaries (harness.cpp:52-57): each block pulls
// `layers` ghost layers of the faces in `axis_mask` from its neighbours'
// current buffers (after their state events), then fills its physical faces.
// Only what the next kernel reads is copied; the ledger
// keeps the reference's full-exchange accounting.
void multi_exchange(ppmlr_gpu_harness* h, int axis_mask, int layers, long step) {
  record_states(h);
  for (size_t r = 0; r < h->blocks.size(); ++r) {
    MK(cudaSetDevice(h->devices[r]));
    for (int face = 0; face < 6; ++face) {
      const int nb = h->plan[r].neighbor[face];
      if (nb < 0 || !((axis_mask >> (face / 2)) & 1)) continue;
      MK(cudaStreamWaitEvent(stream_of(h, r), h->ev_state[nb], 0));
      if (int e = ppmlr_gpu_block_copy_face(h->blocks[r], face, h->blocks[nb], layers))
        throw SpecError(e, ppmlr_gpu_last_error());
    }
    if (int e = ppmlr_gpu_block_fill_boundaries(h->blocks[r], axis_mask, layers))
      throw SpecError(e, ppmlr_gpu_last_error());
  }
  record_exchange(h, step);
}

// The first failure in the reference's order: earliest (step, phase), then
// the lowest rank (its loops run rank by rank), then the block's own key.
// A non-finite CFL candidate of the step after the window is deferred to the
// next advance, like the single-block path (block.cu check_impl).
int multi_check(ppmlr_gpu_harness* h) {
  int best = -1;
  unsigned long long best_key = kNoError, step = 0;
  for (size_t r = 0; r < h->blocks.size(); ++r) {
    unsigned long long key = kNoError;
    if (int e = block_read_error(h->blocks[r], &key, &step)) return e;
    if (key == kNoError) continue;
    if (best < 0 || (key >> kErrAxisShift) < (best_key >> kErrAxisShift)) {
      best = (int)r;
      best_key = key;
    }
  }
  if (best < 0) return 0;
  for (auto* b : h->blocks) {
    block_reset_error(b);
    b->dt_valid = false;
  }
  if (err_phase(best_key) == kPhaseCfl && err_step(best_key) == (step & kErrStepMask)) return 0;
  return block_raise_error(h->blocks[best], best_key);
}

// `steps` Harness::advance steps of a multi-block layout, stream-ordered on
// every block; the dt of the last step is returned in *dt_last.
int multi_run(ppmlr_gpu_harness* h, long steps, double* dt_last) {
  static const int order[2][3] = {{0, 1, 2}, {2, 1, 0}};
  const double cfl = h->o.cfl;
  const int with_sources = h->o.with_sources;
  return guarded([&] {
    // the blocks' local cfl*min, unless the previous window left it for
    // this state (every block; any upload or step outside clears it)
    bool valid = true;
    for (auto* b : h->blocks) valid = valid && b->dt_valid && b->dt_cfl == cfl;
    for (auto* b : h->blocks) {
      if (int e = block_begin_window(b, h->step)) throw SpecError(e, ppmlr_gpu_last_error());
      if (!valid)
        if (int e = ppmlr_gpu_block_local_dt_async(b, cfl))
          throw SpecError(e, ppmlr_gpu_last_error());
    }
    for (long s = 0; s < steps; ++s) {
      const int parity = (h->step + s) % 2 == 0 ? 0 : 1;
      multi_global_dt(h);
      for (int k = 0; k < 3; ++k) {
        const int axis = order[parity][k];
        multi_exchange(h, 1 << axis, kG, h->step + s);
        for (size_t r = 0; r < h->blocks.size(); ++r)
          if (int e = ppmlr_gpu_block_sweep_async(h->blocks[r], axis, k))
            throw SpecError(e, ppmlr_gpu_last_error());
      }
      if (with_sources) multi_exchange(h, 7, 1, h->step + s);
      for (size_t r = 0; r < h->blocks.size(); ++r)
        if (int e = ppmlr_gpu_block_end_step(h->blocks[r], cfl, with_sources))
          throw SpecError(e, ppmlr_gpu_last_error());
    }
    // dt of the last step: block 0's d_dt_prev, host sync
    double dt = 0.0, t = 0.0;
    if (int e = block_last_dt_time(h->blocks[0], &dt, &t))
      throw SpecError(e, ppmlr_gpu_last_error());
    if (int e = multi_check(h)) return e;
    for (auto* b : h->blocks) {  // the fused CFL left the next local cfl*min
      b->dt_valid = true;
      b->dt_cfl = cfl;
    }
    h->step += steps;
    h->time = t;
    if (dt_last) *dt_last = dt;
    return 0;
  });
}

}  // namespace

extern "C" {

int ppmlr_build_axis(const ppmlr_axis_spec* spec, double* edges, double* centers,
                     double* spacings, int cap, int* n_out) {
  return guarded([&] {
    const Axis a = make_axis(*spec);
    *n_out = a.n();
    if (a.n() > cap) invalid("build_axis: output capacity too small");
    std::copy(a.edges.begin(), a.edges.end(), edges);
    std::copy(a.centers.begin(), a.centers.end(), centers);
    std::copy(a.spacings.begin(), a.spacings.end(), spacings);
    return 0;
  });
}

int ppmlr_layout(const ppmlr_axis_spec specs[3], int px, int py, int pz, int* blocks,
                 int cap_blocks, int* nblocks, int* ionosphere_rank) {
  return guarded([&] {
    Axis ax[3] = {make_axis(specs[0]), make_axis(specs[1]), make_axis(specs[2])};
    const int cnt[3] = {px, py, pz};
    const auto plan = plan_layout(cnt, ax, ionosphere_rank);
    *nblocks = (int)plan.size();
    if ((int)plan.size() > cap_blocks) invalid("layout: output capacity too small");
    for (size_t b = 0; b < plan.size(); ++b) {
      int* o = blocks + 16 * b;
      o[0] = plan[b].rank;
      for (int a = 0; a < 3; ++a) {
        o[1 + a] = plan[b].coords[a];
        o[4 + a] = plan[b].lo[a];
        o[7 + a] = plan[b].n[a];
      }
      for (int f = 0; f < 6; ++f) o[10 + f] = plan[b].neighbor[f];
    }
    return 0;
  });
}

int ppmlr_host_block_state(const ppmlr_axis_spec specs[3], int px, int py, int pz,
                           const ppmlr_gpu_options* opts, int rank, int ic_kind,
                           const double* params, double* fields, double* bd,
                           int64_t* frozen_idx, double* frozen_states, int64_t* n_frozen,
                           double* centers_cat, double* spacings_cat) {
  return guarded([&] {
    Axis ax[3] = {make_axis(specs[0]), make_axis(specs[1]), make_axis(specs[2])};
    const int cnt[3] = {px, py, pz};
    int iono = 0;
    const auto plan = plan_layout(cnt, ax, &iono);
    if (rank < 0 || rank >= (int)plan.size()) invalid("no such block");
    if (opts->ghost < 4) invalid("ghost width must be >= 4");
    const HostBlock hb = host_block(ax, plan[rank], opts->ghost);
    std::vector<double> bdv, f, fst;
    std::vector<int64_t> fidx;
    ChunkInit ci;
    ci.hb = &hb;
    ci.o = opts;
    if (ic_kind < 0) {
      ci.kind = -1;
      ci.mp = {params ? params[0] : 1.0, params ? params[1] : 0.1, params ? params[2] : 3.0,
               params ? params[3] : 3.0};
      ci.fidx = &fidx;
      ci.fst = &fst;
    } else {
      ci.kind = ic_kind;
      ci.ic = ic_of(ic_kind, params);
    }
    // straight into the caller's arrays (every cell's 8 values, and its
    // dipole, are written); geometry only when no state is requested
    if (fields) {
      ci(0, hb.n[2] + 2 * hb.g, fields, opts->with_dipole ? bd : nullptr);
    } else if (bd || frozen_idx || frozen_states || n_frozen) {
      block_fill(hb, ci, f, opts->with_dipole ? &bdv : nullptr);
      if (bd && !bdv.empty()) std::copy(bdv.begin(), bdv.end(), bd);
    }
    // *n_frozen > 0 on entry: the capacity of frozen_idx / frozen_states
    if (n_frozen && *n_frozen > 0 && (int64_t)fidx.size() > *n_frozen)
      invalid("host_block_state: frozen-core capacity too small");
    if (frozen_idx) std::copy(fidx.begin(), fidx.end(), frozen_idx);
    if (frozen_states) std::copy(fst.begin(), fst.end(), frozen_states);
    if (n_frozen) *n_frozen = (int64_t)fidx.size();
    size_t off = 0;
    for (int a = 0; a < 3; ++a) {
      if (centers_cat) std::copy(hb.cen[a].begin(), hb.cen[a].end(), centers_cat + off);
      if (spacings_cat) std::copy(hb.spc[a].begin(), hb.spc[a].end(), spacings_cat + off);
      off += hb.cen[a].size();
    }
    return 0;
  });
}

int ppmlr_gpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

long ppmlr_tde_units(int px, int py, int pz) {
  return (long)px * py * (pz - 1) + (long)px * (py - 1) * pz + (long)(px - 1) * py * pz;
}

uint64_t ppmlr_exchanged_bytes(const ppmlr_axis_spec specs[3], int px, int py, int pz,
                               int ghost, int bytes_per_cell) {
  uint64_t total = 0;
  try {
    const long cnt[3] = {px, py, pz};
    const long cells[3] = {make_axis(specs[0]).n(), make_axis(specs[1]).n(),
                           make_axis(specs[2]).n()};
    for (int a = 0; a < 3; ++a) {
      const int b = (a + 1) % 3, c = (a + 2) % 3;
      const uint64_t faces = (uint64_t)(cnt[a] - 1) * cnt[b] * cnt[c];
      const uint64_t face_cells = (uint64_t)(cells[b] / cnt[b]) * (cells[c] / cnt[c]);
      total += faces * face_cells * ghost * bytes_per_cell * 2;
    }
  } catch (const std::exception& e) {
    set_error(e.what());
    return 0;
  }
  return total;
}

int ppmlr_gpu_harness_create(const ppmlr_axis_spec specs[3], int px, int py, int pz,
                             const ppmlr_gpu_options* opts, ppmlr_gpu_harness** out) {
  return ppmlr_gpu_harness_create_on(specs, px, py, pz, opts, &opts->device, 1, out);
}

int ppmlr_gpu_harness_create_on(const ppmlr_axis_spec specs[3], int px, int py, int pz,
                                const ppmlr_gpu_options* opts, const int* devices,
                                int ndevices, ppmlr_gpu_harness** out) {
  *out = nullptr;
  auto* h = new ppmlr_gpu_harness();
  const int rc = guarded([&] {
    if (!devices || ndevices < 1) invalid("create_on: empty device list");
    for (int a = 0; a < 3; ++a) h->ax[a] = make_axis(specs[a]);
    h->cnt[0] = px;
    h->cnt[1] = py;
    h->cnt[2] = pz;
    h->o = *opts;
    if (h->o.ghost < 4) invalid("ghost width must be >= 4");
    h->plan = plan_layout(h->cnt, h->ax, &h->iono);
    if (h->o.boundary == PPMLR_BC_PERIODIC && (px != 1 || py != 1 || pz != 1))
      invalid("periodic boundaries require a (1,1,1) partition");
    const int g = h->g();
    const size_t nb = h->plan.size();
    for (int a = 0; a < 3; ++a) {
      h->cen[a].resize(nb);
      h->spc[a].resize(nb);
    }
    h->fidx.resize(nb);
    h->fst.resize(nb);
    for (size_t r = 0; r < nb; ++r) {
      const BlockPlan& p = h->plan[r];
      for (int a = 0; a < 3; ++a) local_axis(h->ax[a], p.lo[a], p.n[a], g, h->cen[a][r], h->spc[a][r]);
      ppmlr_gpu_block_desc d{};
      for (int a = 0; a < 3; ++a) {
        d.n[a] = p.n[a];
        d.lo[a] = p.lo[a];
        d.centers[a] = h->cen[a][r].data();
        d.spacings[a] = h->spc[a][r].data();
        d.physical[a][0] = p.neighbor[2 * a] < 0;
        d.physical[a][1] = p.neighbor[2 * a + 1] < 0;
      }
      d.ghost = g;
      d.gamma = h->o.gamma;
      d.mu0 = h->o.mu0;
      d.pressure_floor = h->o.pressure_floor;
      d.boundary = h->o.boundary;
      d.wind_rho = h->o.wind_rho;
      d.wind_p = h->o.wind_p;
      for (int a = 0; a < 3; ++a) {
        d.wind_v[a] = h->o.wind_v[a];
        d.wind_imf[a] = h->o.wind_imf[a];
      }
      d.with_dipole = h->o.with_dipole;
      d.precision = h->o.precision;
      d.device = devices[r % ndevices];
      ppmlr_gpu_block* b = nullptr;
      if (int e = ppmlr_gpu_block_create(&d, &b)) throw SpecError(e, ppmlr_gpu_last_error());
      h->blocks.push_back(b);
      h->devices.push_back(d.device);
      // make_block's default state {1, 0, 0, 1} and its dipole
      if (use_device_init(-2)) {
        init_device(h, (int)r, -2, nullptr, true);
      } else {
        ChunkInit ci;
        ci.kind = -2;
        upload_init(h, (int)r, ci, true);
      }
    }
    if (nb > 1) multi_setup(h);
    return 0;
  });
  if (rc) {
    ppmlr_gpu_harness_destroy(h);
    return rc;
  }
  *out = h;
  return 0;
}

void ppmlr_gpu_harness_destroy(ppmlr_gpu_harness* h) {
  if (!h) return;
  if (h->snap_writer.joinable()) h->snap_writer.join();
  for (size_t r = 0; r < h->ev_state.size(); ++r) {
    cudaSetDevice(h->devices[r]);
    cudaEventDestroy(h->ev_state[r]);
  }
  if (!h->devices.empty()) cudaSetDevice(h->devices[0]);
  if (h->ev_dt) cudaEventDestroy(h->ev_dt);
  if (h->d_slots) cudaFree(h->d_slots);
  for (auto* b : h->blocks) ppmlr_gpu_block_destroy(b);
  delete h;
}

int ppmlr_gpu_harness_init_magnetosphere(ppmlr_gpu_harness* h, double rho_core, double p_core,
                                         double falloff, double r_ref) {
  return guarded([&] {
    for (size_t r = 0; r < h->blocks.size(); ++r) {
      ChunkInit ci;
      ci.kind = -1;
      ci.mp = {rho_core, p_core, falloff, r_ref};
      upload_init(h, (int)r, ci, false);
    }
    return 0;
  });
}

int ppmlr_gpu_harness_init_ic(ppmlr_gpu_harness* h, int kind, const double* params) {
  return guarded([&] {
    for (size_t r = 0; r < h->blocks.size(); ++r) {
      if (use_device_init(kind)) {
        init_device(h, (int)r, kind, params, false);
        continue;
      }
      ChunkInit ci;
      ci.kind = kind;
      ci.ic = ic_of(kind, params);
      upload_init(h, (int)r, ci, false);
    }
    return 0;
  });
}

int ppmlr_gpu_harness_set_state(ppmlr_gpu_harness* h, const double* all) {
  return guarded([&] {
    size_t off = 0;
    for (size_t r = 0; r < h->blocks.size(); ++r) {
      h->fidx[r].clear();
      h->fst[r].clear();
      if (int e = ppmlr_gpu_block_upload(h->blocks[r], all + off, nullptr, nullptr, nullptr, 0))
        throw SpecError(e, ppmlr_gpu_last_error());
      off += h->cells(r) * 8;
    }
    return 0;
  });
}

int ppmlr_gpu_harness_compute_dt(ppmlr_gpu_harness* h, double* dt_out) {
  double dt = INFINITY;
  for (auto* b : h->blocks) {
    double d;
    if (int rc = ppmlr_gpu_block_compute_dt(b, h->o.cfl, &d)) return rc;
    dt = std::min(dt, d);
  }
  *dt_out = dt;
  return 0;
}

int ppmlr_gpu_harness_advance(ppmlr_gpu_harness* h, double* dt_out) {
  double dt = 0.0;
  if (h->blocks.size() == 1) {
    // whole-domain block: the fused, graph-captured device step
    if (int rc = ppmlr_gpu_block_advance(h->blocks[0], h->o.cfl, h->o.with_sources, h->step,
                                         &dt))
      return rc;
    for (int e = 0; e < 3 + (h->o.with_sources ? 1 : 0); ++e) record_exchange(h, h->step);
    h->step += 1;
    h->time += dt;
  } else {
    if (int rc = multi_run(h, 1, &dt)) return rc;
  }
  if (dt_out) *dt_out = dt;
  return 0;
}

int ppmlr_gpu_harness_run(ppmlr_gpu_harness* h, long steps) {
  if (h->blocks.size() == 1) {
    double t = h->time;
    if (int rc = ppmlr_gpu_block_run(h->blocks[0], h->o.cfl, h->o.with_sources, h->step, steps,
                                     &t))
      return rc;
    h->time = t;
    for (long s = 0; s < steps; ++s)
      for (int e = 0; e < 3 + (h->o.with_sources ? 1 : 0); ++e) record_exchange(h, h->step + s);
    h->step += steps;
    return 0;
  }
  for (long done = 0; done < steps;) {
    const long k = std::min(steps - done, kMaxStepsPerCheck);
    if (int rc = multi_run(h, k, nullptr)) return rc;
    done += k;
  }
  return 0;
}

int ppmlr_gpu_harness_gather(ppmlr_gpu_harness* h, double* out) {
  const int nx = h->ax[0].n(), ny = h->ax[1].n();
  for (size_t r = 0; r < h->blocks.size(); ++r) {
    const BlockPlan& p = h->plan[r];
    std::vector<double> loc((size_t)p.n[0] * p.n[1] * p.n[2] * 8);
    if (int rc = ppmlr_gpu_block_download_interior(h->blocks[r], loc.data())) return rc;
    for (int k = 0; k < p.n[2]; ++k)
      for (int j = 0; j < p.n[1]; ++j)
        for (int i = 0; i < p.n[0]; ++i) {
          const size_t gi = (size_t)(p.lo[0] + i) +
                            (size_t)nx * ((p.lo[1] + j) + (size_t)ny * (p.lo[2] + k));
          std::memcpy(out + 8 * gi, &loc[8 * ((size_t)i + (size_t)p.n[0] * (j + (size_t)p.n[1] * k))],
                      64);
        }
  }
  return 0;
}

long ppmlr_gpu_harness_step_count(ppmlr_gpu_harness* h) { return h->step; }
double ppmlr_gpu_harness_time(ppmlr_gpu_harness* h) { return h->time; }
int ppmlr_gpu_harness_block_count(ppmlr_gpu_harness* h) { return (int)h->blocks.size(); }
ppmlr_gpu_block* ppmlr_gpu_harness_block(ppmlr_gpu_harness* h, int rank) {
  return rank >= 0 && rank < (int)h->blocks.size() ? h->blocks[rank] : nullptr;
}

void ppmlr_gpu_harness_ledger(ppmlr_gpu_harness* h, uint64_t* bytes, long* messages,
                              long* copy_events) {
  if (bytes) *bytes = h->ledger_bytes;
  if (messages) *messages = h->ledger_messages;
  if (copy_events) *copy_events = h->ledger_events;
}

long ppmlr_gpu_harness_ledger_entries(ppmlr_gpu_harness* h, long* step, int* transport,
                                      long* messages, uint64_t* bytes, long* copy_events,
                                      long max) {
  const long n = (long)h->ledger.size();
  for (long i = 0; i < std::min(n, max); ++i) {
    const LedgerRow& e = h->ledger[i];
    if (step) step[i] = e.step;
    if (transport) transport[i] = e.transport;
    if (messages) messages[i] = e.messages;
    if (bytes) bytes[i] = e.bytes;
    if (copy_events) copy_events[i] = e.copy_events;
  }
  return n;
}

// write_snapshot (snapshot.cpp:58-85) of make_snapshot (ppmlr_main.cpp:20-31):
// "PPLR", u32 version 1, u32 dims[3], u32 ghost, f64 time, u64 step, the
// global edge arrays, the tag "rvvvbbbp", then per field the global
// interior array, x fastest.  Every block's capture is drained plane-chunk
// by plane-chunk into one pinned global chunk and appended to the file.
int ppmlr_gpu_harness_snapshot_begin(ppmlr_gpu_harness* h, const char* path) {
  if (int rc = ppmlr_gpu_harness_snapshot_wait(h)) return rc;
  for (auto* b : h->blocks)
    if (int rc = ppmlr_gpu_block_snapshot_capture(b)) return rc;
  struct Header {
    uint32_t dims[3], ghost;
    double time;
    uint64_t step;
  } hd{{(uint32_t)h->ax[0].n(), (uint32_t)h->ax[1].n(), (uint32_t)h->ax[2].n()},
       (uint32_t)h->o.ghost, h->time, (uint64_t)h->step};
  const std::string file = path;
  h->snap_rc = 0;
  h->snap_err.clear();
  h->snap_writer = std::thread([h, hd, file] {
    auto fail = [&](int rc, const std::string& m) {
      h->snap_rc = rc;
      h->snap_err = m;
    };
    cudaSetDevice(h->o.device);
    FILE* out = std::fopen(file.c_str(), "wb");
    if (!out) return fail(PPMLR_INVALID_SPEC, "snapshot: cannot open for writing: " + file);
    const uint32_t version = 1;
    bool ok = std::fwrite("PPLR", 1, 4, out) == 4 && std::fwrite(&version, 4, 1, out) == 1 &&
              std::fwrite(hd.dims, 4, 3, out) == 3 && std::fwrite(&hd.ghost, 4, 1, out) == 1 &&
              std::fwrite(&hd.time, 8, 1, out) == 1 && std::fwrite(&hd.step, 8, 1, out) == 1;
    for (int a = 0; a < 3 && ok; ++a)
      ok = std::fwrite(h->ax[a].edges.data(), 8, h->ax[a].edges.size(), out) ==
           h->ax[a].edges.size();
    ok = ok && std::fwrite("rvvvbbbp", 1, 8, out) == 8;
    const size_t nx = hd.dims[0], ny = hd.dims[1], nz = hd.dims[2];
    const size_t plane = nx * ny;
    const size_t kchunk = std::max<size_t>(1, std::min<size_t>(nz, (64u << 20) / (plane * 8)));
    double* buf = nullptr;
    if (ok && cudaMallocHost(&buf, plane * kchunk * sizeof(double)) != cudaSuccess) {
      std::fclose(out);
      return fail(PPMLR_RUNTIME, "snapshot: pinned staging allocation failed");
    }
    for (int f = 0; f < 8 && ok; ++f)
      for (size_t k0 = 0; k0 < nz && ok; k0 += kchunk) {
        const size_t nk = std::min(kchunk, nz - k0);
        for (size_t r = 0; r < h->blocks.size(); ++r) {
          const BlockPlan& p = h->plan[r];
          const long lo = std::max<long>(p.lo[2], (long)k0);
          const long hi = std::min<long>(p.lo[2] + p.n[2], (long)(k0 + nk));
          if (lo >= hi) continue;
          double* dst = buf + (size_t)(lo - (long)k0) * plane + (size_t)p.lo[1] * nx + p.lo[0];
          if (int rc = ppmlr_gpu_block_snapshot_read(h->blocks[r], f, (int)(lo - p.lo[2]),
                                                     (int)(hi - lo), dst, (int64_t)nx,
                                                     (int64_t)plane)) {
            cudaFreeHost(buf);
            std::fclose(out);
            return fail(rc, ppmlr_gpu_last_error());
          }
        }
        ok = std::fwrite(buf, 8, plane * nk, out) == plane * nk;
      }
    if (buf) cudaFreeHost(buf);
    if (std::fclose(out) != 0) ok = false;
    if (!ok) fail(PPMLR_INVALID_SPEC, "snapshot: write failed: " + file);
  });
  return 0;
}

int ppmlr_gpu_harness_snapshot_wait(ppmlr_gpu_harness* h) {
  if (h->snap_writer.joinable()) h->snap_writer.join();
  const int rc = h->snap_rc;
  if (rc) set_error(h->snap_err);
  h->snap_rc = 0;
  return rc;
}

int ppmlr_gpu_harness_snapshot(ppmlr_gpu_harness* h, const char* path) {
  if (int rc = ppmlr_gpu_harness_snapshot_begin(h, path)) return rc;
  return ppmlr_gpu_harness_snapshot_wait(h);
}

int64_t ppmlr_gpu_harness_frozen(ppmlr_gpu_harness* h, int rank, int64_t* idx, double* states) {
  const auto& fi = h->fidx[rank];
  if (idx) std::copy(fi.begin(), fi.end(), idx);
  if (states) std::copy(h->fst[rank].begin(), h->fst[rank].end(), states);
  return (int64_t)fi.size();
}

int ppmlr_gpu_harness_block_geometry(ppmlr_gpu_harness* h, int rank, int* n, int* lo,
                                     double* centers_cat, double* spacings_cat, double* bd) {
  if (rank < 0 || rank >= (int)h->blocks.size()) {
    set_error("no such block");
    return PPMLR_INVALID_SPEC;
  }
  const BlockPlan& p = h->plan[rank];
  size_t off = 0;
  for (int a = 0; a < 3; ++a) {
    n[a] = p.n[a];
    lo[a] = p.lo[a];
    if (centers_cat) std::copy(h->cen[a][rank].begin(), h->cen[a][rank].end(), centers_cat + off);
    if (spacings_cat)
      std::copy(h->spc[a][rank].begin(), h->spc[a][rank].end(), spacings_cat + off);
    off += h->cen[a][rank].size();
  }
  if (bd && h->o.with_dipole) {
    std::vector<double> bdv;
    block_dipole(host_block(h->ax, p, h->g()), h->o.mu0, bdv);
    std::copy(bdv.begin(), bdv.end(), bd);
  }
  return 0;
}

}  // extern "C"
