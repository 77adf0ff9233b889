// C-ABI shim over the unmodified reference sources.  TEST INFRASTRUCTURE ONLY
// (see ref_shim.h).  Built by oracle/Makefile together with
// /root/reference/proj/src/*.cpp into oracle/_ref/libppmlr_ref.so; this file
// is the only piece of that library that lives in this repository.
#include "ref_shim.h"

#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "ppmlr/decomp.hpp"
#include "ppmlr/errors.hpp"
#include "ppmlr/grid.hpp"
#include "ppmlr/harness.hpp"
#include "ppmlr/snapshot.hpp"
#include "ppmlr/ppm1d.hpp"
#include "ppmlr/stepper.hpp"
#include "ppmlr/verify.hpp"

using namespace ppmlr;

namespace {

void put_err(char* err, int errlen, const char* msg) {
  if (err && errlen > 0) {
    std::strncpy(err, msg, errlen - 1);
    err[errlen - 1] = 0;
  }
}

template <typename F>
int guarded(char* err, int errlen, F&& f) {
  try {
    f();
    return 0;
  } catch (const InvalidSpec& e) {
    put_err(err, errlen, e.what());
    return 1;
  } catch (const UnphysicalState& e) {
    put_err(err, errlen, e.what());
    return 2;
  } catch (const StepRejected& e) {
    put_err(err, errlen, e.what());
    return 3;
  } catch (const OutOfRange& e) {
    put_err(err, errlen, e.what());
    return 4;
  } catch (const Error& e) {
    put_err(err, errlen, e.what());
    return 5;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 6;
  }
}

AxisSpec to_spec(const ref_axis_spec& s) {
  return {s.min, s.max, s.uniform_lo, s.uniform_hi, s.d_uniform, s.cells, s.ratio};
}

StretchedGrid make_grid(const ref_axis_spec* s) {
  return {build_axis(to_spec(s[0])), build_axis(to_spec(s[1])), build_axis(to_spec(s[2]))};
}

HarnessOptions to_opts(const ref_options& o) {
  HarnessOptions h;
  h.cfl = o.cfl;
  h.ghost = o.ghost;
  h.boundary = o.boundary == 0   ? BoundaryMode::Outflow
               : o.boundary == 1 ? BoundaryMode::Periodic
                                 : BoundaryMode::Magnetosphere;
  h.transport = o.transport == 0 ? TransportKind::Staged : TransportKind::Direct;
  h.with_sources = o.with_sources != 0;
  h.with_dipole = o.with_dipole != 0;
  h.wind.rho_sw = o.wind_rho;
  h.wind.p_sw = o.wind_p;
  h.wind.v_sw = {o.wind_v[0], o.wind_v[1], o.wind_v[2]};
  h.wind.imf = {o.wind_imf[0], o.wind_imf[1], o.wind_imf[2]};
  h.constants.mu0 = o.mu0;
  h.constants.gamma = o.gamma;
  h.constants.pressure_floor = o.pressure_floor;
  return h;
}

void state_to(const PrimitiveState& s, double* o) {
  o[0] = s.rho;
  o[1] = s.v.x;
  o[2] = s.v.y;
  o[3] = s.v.z;
  o[4] = s.bprime.x;
  o[5] = s.bprime.y;
  o[6] = s.bprime.z;
  o[7] = s.p;
}

PrimitiveState state_from(const double* i) {
  PrimitiveState s;
  s.rho = i[0];
  s.v = {i[1], i[2], i[3]};
  s.bprime = {i[4], i[5], i[6]};
  s.p = i[7];
  return s;
}

// The synthetic initial conditions of the benchmark configurations
// (BASELINE.json configs).  The product's host code
// implements the same formulas; tests/golden pins both to each other.
std::function<PrimitiveState(const Vec3&)> make_ic(int kind, const double* p) {
  switch (kind) {
    case 0: {
      const PrimitiveState s = state_from(p);
      return [s](const Vec3&) { return s; };
    }
    case 1:
      return [](const Vec3& r) {
        PrimitiveState q;
        const bool left = r.x < 0.5;
        q.rho = left ? 1.0 : 0.125;
        q.p = left ? 1.0 : 0.1;
        q.bprime = {0.75, left ? 1.0 : -1.0, 0.0};
        return q;
      };
    case 2: {
      const double g = p[0];
      return [g](const Vec3& r) {
        PrimitiveState q;
        q.rho = g * g;
        q.p = g;
        q.v = {-std::sin(r.y), std::sin(r.x), 0.0};
        q.bprime = {-std::sin(r.y), std::sin(2.0 * r.x), 0.0};
        return q;
      };
    }
    case 3: {
      const double p_in = p[0], p_out = p[1], rad = p[2];
      return [=](const Vec3& r) {
        PrimitiveState q;
        const double cx = std::floor(r.x + 0.5);
        const double dx = r.x - cx;
        const double r2 = dx * dx + r.y * r.y + r.z * r.z;
        q.rho = 1.0;
        q.p = r2 < rad * rad ? p_in : p_out;
        q.bprime = {std::sqrt(0.5), std::sqrt(0.5), 0.0};
        return q;
      };
    }
    case 4:
      return [](const Vec3& r) {
        const double w = std::exp(-norm2(r) / 2.0);
        PrimitiveState q;
        q.rho = 1.0 + 0.3 * w;
        q.v = Vec3{-r.y, r.x, 0.0} * (0.2 * w);
        q.bprime = Vec3{-r.y, r.x, 0.1} * 0.1;
        q.p = 1.0 + 0.2 * w;
        return q;
      };
    case 5:
      return [](const Vec3& r) {
        const double w = std::exp(-0.5 * dot(r, r));
        return PrimitiveState{1.0 + 0.3 * w,
                              {0.2 * w * -r.y, 0.2 * w * r.x, 0.0},
                              {0.1 * -r.y, 0.1 * r.x, 0.01},
                              1.0 + 0.2 * w};
      };
    case 6:
      return [](const Vec3& r) {
        PrimitiveState q;
        q.rho = 1.0;
        q.p = 0.1 + 5.0 * std::exp(-norm2(r) / (0.25 * 0.25));
        return q;
      };
    default:
      throw InvalidSpec("ref_shim: unknown IC kind " + std::to_string(kind));
  }
}

struct Handle {
  Harness h;
};

Harness& H(void* h) { return static_cast<Handle*>(h)->h; }
BlockState& B(void* h, int r) { return const_cast<BlockState&>(H(h).block(r)); }

}  // namespace

extern "C" {

int ref_build_axis(const ref_axis_spec* spec, double* edges, double* centers,
                   double* spacings, int cap, int* n_out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const Axis a = build_axis(to_spec(*spec));
    *n_out = a.n();
    if (a.n() > cap) throw InvalidSpec("ref_build_axis: capacity too small");
    for (int i = 0; i <= a.n(); ++i) edges[i] = a.edges[i];
    for (int i = 0; i < a.n(); ++i) {
      centers[i] = a.centers[i];
      spacings[i] = a.spacings[i];
    }
  });
}

int ref_sweep_1d(double* states, const double* bd, const double* spacings, int n,
                 int ghost, double dt, int dir, double gamma, double mu0,
                 double pressure_floor, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    Strip1D s;
    s.n = n;
    s.ghost = ghost;
    const int nn = s.total();
    s.spacings.assign(spacings, spacings + nn);
    s.states.resize(nn);
    for (int i = 0; i < nn; ++i) s.states[i] = state_from(states + 8 * i);
    if (bd) {
      s.bd.resize(nn);
      for (int i = 0; i < nn; ++i) s.bd[i] = {bd[3 * i], bd[3 * i + 1], bd[3 * i + 2]};
    }
    Constants c;
    c.gamma = gamma;
    c.mu0 = mu0;
    c.pressure_floor = pressure_floor;
    sweep_1d(s, dt, dir, c);
    for (int i = 0; i < nn; ++i) state_to(s.states[i], states + 8 * i);
  });
}

double ref_strip_max_dt(const double* states, const double* bd, const double* spacings,
                        int n, int ghost, int dir, double gamma, double mu0) {
  Strip1D s;
  s.n = n;
  s.ghost = ghost;
  const int nn = s.total();
  s.spacings.assign(spacings, spacings + nn);
  s.states.resize(nn);
  for (int i = 0; i < nn; ++i) s.states[i] = state_from(states + 8 * i);
  if (bd) {
    s.bd.resize(nn);
    for (int i = 0; i < nn; ++i) s.bd[i] = {bd[3 * i], bd[3 * i + 1], bd[3 * i + 2]};
  }
  Constants c;
  c.gamma = gamma;
  c.mu0 = mu0;
  return strip_max_dt(s, dir, c);
}

int ref_layout(const ref_axis_spec* specs3, int px, int py, int pz, int* blocks,
               int cap_blocks, int* nblocks, int* iono_rank, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const StretchedGrid g = make_grid(specs3);
    const BlockLayout l = layout({px, py, pz}, g);
    *nblocks = static_cast<int>(l.blocks.size());
    *iono_rank = l.ionosphere_rank;
    if (*nblocks > cap_blocks) throw InvalidSpec("ref_layout: capacity too small");
    for (int b = 0; b < *nblocks; ++b) {
      const BlockInfo& i = l.blocks[b];
      int* o = blocks + 16 * b;
      o[0] = i.rank;
      for (int a = 0; a < 3; ++a) {
        o[1 + a] = i.coords[a];
        o[4 + a] = i.lo[a];
        o[7 + a] = i.n[a];
      }
      for (int f = 0; f < 6; ++f) o[10 + f] = i.neighbor[f];
    }
  });
}

void* ref_harness_create(const ref_axis_spec* specs3, int px, int py, int pz,
                         const ref_options* opts, char* err, int errlen) {
  Handle* out = nullptr;
  guarded(err, errlen, [&] {
    const StretchedGrid g = make_grid(specs3);
    out = new Handle{Harness(g, layout({px, py, pz}, g), to_opts(*opts))};
  });
  return out;
}

void ref_harness_destroy(void* h) { delete static_cast<Handle*>(h); }

int ref_harness_block_count(void* h) { return H(h).block_count(); }

void ref_harness_block_dims(void* h, int r, int* n, int* lo, int* ghost) {
  const BlockState& b = H(h).block(r);
  for (int a = 0; a < 3; ++a) {
    n[a] = b.n[a];
    lo[a] = b.lo[a];
  }
  *ghost = b.ghost;
}

void ref_harness_block_axis(void* h, int r, int a, double* centers, double* spacings) {
  const BlockState& b = H(h).block(r);
  for (int i = 0; i < b.span(a); ++i) {
    centers[i] = b.centers[a][i];
    spacings[i] = b.spacings[a][i];
  }
}

void ref_harness_get_fields(void* h, int r, double* out) {
  const BlockState& b = H(h).block(r);
  for (std::size_t i = 0; i < b.fields.size(); ++i) state_to(b.fields[i], out + 8 * i);
}

void ref_harness_set_fields(void* h, int r, const double* in) {
  BlockState& b = B(h, r);
  for (std::size_t i = 0; i < b.fields.size(); ++i) b.fields[i] = state_from(in + 8 * i);
}

void ref_harness_get_bd(void* h, int r, double* out) {
  const BlockState& b = H(h).block(r);
  for (std::size_t i = 0; i < b.bd.size(); ++i) {
    out[3 * i] = b.bd[i].x;
    out[3 * i + 1] = b.bd[i].y;
    out[3 * i + 2] = b.bd[i].z;
  }
}

int64_t ref_harness_frozen_count(void* h, int r) {
  return static_cast<int64_t>(H(h).block(r).frozen_core.size());
}

void ref_harness_get_frozen(void* h, int r, int64_t* idx, double* states) {
  const BlockState& b = H(h).block(r);
  for (std::size_t i = 0; i < b.frozen_core.size(); ++i) {
    idx[i] = b.frozen_core[i].first;
    state_to(b.frozen_core[i].second, states + 8 * i);
  }
}

int ref_harness_init_magnetosphere(void* h, double rho_core, double p_core,
                                   double falloff, double r_ref, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    InitialProfiles p;
    p.rho_core = rho_core;
    p.p_core = p_core;
    p.falloff = falloff;
    p.r_ref = r_ref;
    H(h).init_magnetosphere(p);
  });
}

int ref_harness_init_ic(void* h, int kind, const double* params, char* err, int errlen) {
  return guarded(err, errlen, [&] { H(h).init_with(make_ic(kind, params)); });
}

int ref_harness_advance(void* h, double* dt_out, char* err, int errlen) {
  return guarded(err, errlen, [&] { *dt_out = H(h).advance(); });
}

int ref_harness_compute_dt(void* h, double* dt_out, char* err, int errlen) {
  return guarded(err, errlen, [&] { *dt_out = H(h).compute_global_dt(); });
}

void ref_harness_gather(void* h, double* out) {
  const auto v = H(h).gather_interior();
  for (std::size_t i = 0; i < v.size(); ++i) state_to(v[i], out + 8 * i);
}

long ref_harness_step(void* h) { return H(h).step_count(); }
double ref_harness_time(void* h) { return H(h).time(); }
uint64_t ref_harness_ledger_bytes(void* h) { return H(h).ledger().total_bytes; }
long ref_harness_ledger_messages(void* h) { return H(h).ledger().total_messages; }
long ref_harness_ledger_copy_events(void* h) { return H(h).ledger().total_copy_events; }

// The reference's ledger entries (TransferLedger::entries, exchange.hpp:40-61);
// returns the count, fills at most `max`.  (The CSV text is formatted by the
// caller: ostream number formatting inside a ctypes-loaded library crashed
// in the Python test process.)
long ref_harness_ledger_entries(void* h, long* step, int* transport, long* messages,
                                uint64_t* bytes, long* copy_events, long max) {
  const auto& e = H(h).ledger().entries;
  const long n = (long)e.size();
  for (long i = 0; i < std::min(n, max); ++i) {
    step[i] = e[i].step;
    transport[i] = e[i].transport == TransportKind::Direct ? 1 : 0;
    messages[i] = e[i].messages;
    bytes[i] = e[i].bytes;
    copy_events[i] = e[i].copy_events;
  }
  return n;
}

// run_suite (verify.cpp:234-243): metrics and pass flags of one suite.
int ref_run_suite(const char* name, double* metrics, int* pass, int max, char* err,
                  int errlen) {
  int n = 0;
  const int rc = guarded(err, errlen, [&] {
    const auto res = run_suite(name);
    for (const auto& r : res) {
      if (n < max) {
        metrics[n] = r.metric;
        pass[n] = r.pass ? 1 : 0;
      }
      ++n;
    }
  });
  return rc ? -rc : n;
}

// `ppmlr run`'s snapshot of the current state: make_snapshot
// (tools/ppmlr_main.cpp:20-31) + write_snapshot (snapshot.cpp:58-85).
int ref_harness_write_snapshot(void* h, const char* path, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const Harness& hh = H(h);
    Snapshot s;
    const StretchedGrid& g = hh.grid();
    s.dims = {static_cast<std::uint32_t>(g.x.n()), static_cast<std::uint32_t>(g.y.n()),
              static_cast<std::uint32_t>(g.z.n())};
    s.ghost = static_cast<std::uint32_t>(hh.options().ghost);
    s.time = hh.time();
    s.step = static_cast<std::uint64_t>(hh.step_count());
    for (int a = 0; a < 3; ++a) s.edges[a] = g.axis(a).edges;
    s.fields = hh.gather_interior();
    write_snapshot(path, s);
  });
}

int ref_bench(const ref_axis_spec* specs3, const ref_options* opts, int ic_kind,
              const double* ic_params, int threads, int steps, double* rate,
              double* seconds, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const StretchedGrid g = make_grid(specs3);
    const BlockLayout l = layout({1, 1, 1}, g);
    const HarnessOptions o = to_opts(*opts);
    std::vector<Harness> hs;
    hs.reserve(threads);
    for (int t = 0; t < threads; ++t) {
      hs.emplace_back(g, l, o);
      if (ic_kind < 0)
        hs.back().init_magnetosphere(InitialProfiles{});
      else
        hs.back().init_with(make_ic(ic_kind, ic_params));
    }
    std::vector<double> secs(threads, 0.0);
    std::vector<std::string> errs(threads);
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        try {
          const auto t0 = std::chrono::steady_clock::now();
          hs[t].run(steps);
          secs[t] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0)
                        .count();
        } catch (const std::exception& e) {
          errs[t] = e.what();
        }
      });
    for (auto& th : pool) th.join();
    for (const auto& e : errs)
      if (!e.empty()) throw Error(e);
    double worst = 0.0;
    for (double s : secs) worst = std::max(worst, s);
    const double cells = static_cast<double>(g.x.n()) * g.y.n() * g.z.n();
    *seconds = worst;
    *rate = cells * steps * threads / worst;
  });
}

}  // extern "C"
