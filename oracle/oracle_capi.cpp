// TEST INFRASTRUCTURE ONLY — flat C ABI over the CPU oracle (tlsph_oracle.hpp)
// so pytest and bench.py can drive it through ctypes. Never linked by the
// product library. Arrays cross the boundary in reference particle order,
// vectors as n*D doubles, matrices as n*D*D doubles (row-major per particle).
#include <chrono>
#include <cstdio>
#include <memory>
#include <type_traits>
#include <variant>

#include "tlsph_oracle.hpp"

namespace {

thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    g_err.clear();
    return 0;
  } catch (const orc::Error& e) {
    g_err = e.what();
    return static_cast<int>(e.kind);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 7;
  }
}

template <int D>
struct Sim {
  static constexpr int dim = D;
  orc::ParticleSystem<D> sys;
  orc::CellGrid<D> grid;
  std::vector<std::vector<int>> blocks;
  orc::Neighborhood<D> nbh;
  orc::ExternalAccel<D> ext;
  orc::Material mat;
  double h = 0.0;
  // loop state kept for a resumed run (orc_run with params[10] != 0): the damping stream, t, counts
  std::unique_ptr<orc::RandomSource> loop_rng;
  double loop_t = 0.0;
  long long loop_steps = 0, loop_damped = 0;
};

struct Handle {
  int dim = 0;
  std::unique_ptr<Sim<2>> s2;
  std::unique_ptr<Sim<3>> s3;
};

template <typename Fn>
void with_sim(void* hv, Fn&& fn) {
  auto* h = static_cast<Handle*>(hv);
  orc::require(h != nullptr, orc::ErrorKind::InvalidArgument, "null oracle handle");
  if (h->dim == 2) fn(*h->s2);
  else fn(*h->s3);
}

// field ids shared with tests/oracle.py
enum Field { R0 = 0, R = 1, V = 2, A = 3, F = 4, DFDT = 5, B0 = 6, V0 = 7, M = 8, RHO0 = 9, RHO = 10,
             BODY = 11, CONSTRAINED = 12 };

template <int D>
void copy_field(Sim<D>& s, int field, double* out, const double* in) {
  auto& p = s.sys;
  const std::size_t n = p.size();
  auto vec = [&](std::vector<orc::Vec<D>>& a) {
    if (out) for (std::size_t i = 0; i < n; ++i) for (int d = 0; d < D; ++d) out[i * D + d] = a[i][d];
    if (in) { a.resize(n); for (std::size_t i = 0; i < n; ++i) for (int d = 0; d < D; ++d) a[i][d] = in[i * D + d]; }
  };
  auto mat = [&](std::vector<orc::Mat<D>>& a) {
    if (out) for (std::size_t i = 0; i < n; ++i) for (int r = 0; r < D; ++r) for (int c = 0; c < D; ++c) out[(i * D + r) * D + c] = a[i](r, c);
    if (in) for (std::size_t i = 0; i < n; ++i) for (int r = 0; r < D; ++r) for (int c = 0; c < D; ++c) a[i](r, c) = in[(i * D + r) * D + c];
  };
  auto sc = [&](std::vector<double>& a) {
    if (out) for (std::size_t i = 0; i < n; ++i) out[i] = a[i];
    if (in) for (std::size_t i = 0; i < n; ++i) a[i] = in[i];
  };
  switch (field) {
    case R0: vec(p.r0); break;
    case R: vec(p.r); break;
    case V: vec(p.v); break;
    case A: vec(p.a); break;
    case F: mat(p.F); break;
    case DFDT: mat(p.dFdt); break;
    case B0: mat(p.B0); break;
    case V0: sc(p.V0); break;
    case M: sc(p.m); break;
    case RHO0: sc(p.rho0); break;
    case RHO: sc(p.rho); break;
    case BODY:
      if (out) { if (s.ext.body.empty()) std::fill(out, out + n * D, 0.0); else vec(s.ext.body); }
      if (in) vec(s.ext.body);
      break;
    case CONSTRAINED:
      if (out) for (std::size_t i = 0; i < n; ++i) out[i] = p.constrained[i];
      if (in) for (std::size_t i = 0; i < n; ++i) p.constrained[i] = in[i] != 0.0 ? 1 : 0;
      break;
    default: throw orc::Error(orc::ErrorKind::InvalidArgument, "unknown field id");
  }
}

template <int D>
std::unique_ptr<Sim<D>> make_sim(std::size_t n, const double* r0, const double* V0, const double* rho0,
                                 const unsigned char* constrained, double h, int build) {
  auto s = std::make_unique<Sim<D>>();
  s->h = h;
  for (std::size_t i = 0; i < n; ++i) {
    orc::Vec<D> p;
    for (int d = 0; d < D; ++d) p[d] = r0[i * D + d];
    s->sys.add_particle(p, V0[i], rho0[i]);
    if (constrained) s->sys.constrained[i] = constrained[i];
  }
  if (build) {
    const orc::SmoothingKernel kernel(h, D);
    s->grid = orc::build_cell_grid<D>(s->sys.r0, kernel.support_radius());
    s->blocks = orc::block_decompose<D>(s->grid);
    s->nbh = orc::build_reference_neighborhoods<D>(s->sys.r0, s->sys.V0, kernel, s->grid);
  }
  return s;
}

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_openmp_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

// Creates an oracle system; build=1 runs build_cell_grid + block_decompose +
// build_reference_neighborhoods with cutoff 2h (runner.cpp:299-305).
int orc_create(int dim, size_t n, const double* r0, const double* V0, const double* rho0,
               const unsigned char* constrained, double h, int build, void** out) {
  *out = nullptr;
  return guarded([&] {
    orc::require(dim == 2 || dim == 3, orc::ErrorKind::InvalidArgument, "dimension must be 2 or 3");
    auto hd = std::make_unique<Handle>();
    hd->dim = dim;
    if (dim == 2) hd->s2 = make_sim<2>(n, r0, V0, rho0, constrained, h, build);
    else hd->s3 = make_sim<3>(n, r0, V0, rho0, constrained, h, build);
    *out = hd.release();
  });
}

void orc_destroy(void* h) { delete static_cast<Handle*>(h); }

size_t orc_size(void* hv) {
  size_t n = 0;
  guarded([&] { with_sim(hv, [&](auto& s) { n = s.sys.size(); }); });
  return n;
}

int orc_set_field(void* hv, int field, const double* in) {
  return guarded([&] { with_sim(hv, [&](auto& s) { copy_field(s, field, nullptr, in); }); });
}

int orc_get_field(void* hv, int field, double* out) {
  return guarded([&] { with_sim(hv, [&](auto& s) { copy_field(s, field, out, nullptr); }); });
}

int orc_set_material(void* hv, double E, double nu, double rho0, int model) {
  return guarded([&] {
    with_sim(hv, [&](auto& s) {
      s.mat = orc::material_from_young_poisson(E, nu, rho0, model == 1 ? orc::Model::NeoHookean : orc::Model::LinearKirchhoff);
    });
  });
}

// out: [lambda, mu, K, G, E, nu, rho0, c]
int orc_material(double E, double nu, double rho0, int model, double* out) {
  return guarded([&] {
    const auto m = orc::material_from_young_poisson(E, nu, rho0, model == 1 ? orc::Model::NeoHookean : orc::Model::LinearKirchhoff);
    const double v[8] = {m.lambda, m.mu, m.K, m.G, m.E, m.nu, m.rho0, m.c};
    std::copy(v, v + 8, out);
  });
}

// ---- grid / blocks / neighbourhood queries
// dims_out[D], origin_out[D], cell_size_out, ncells
int orc_grid_info(void* hv, int* dims_out, double* origin_out, double* cell_size_out, long long* ncells_out) {
  return guarded([&] {
    with_sim(hv, [&](auto& s) {
      constexpr int D = std::remove_reference_t<decltype(s)>::dim;
      for (int d = 0; d < D; ++d) { dims_out[d] = s.grid.dims[d]; origin_out[d] = s.grid.origin[d]; }
      *cell_size_out = s.grid.cell_size;
      *ncells_out = s.grid.cell_count();
    });
  });
}

// cell_of[n]; cell_start[ncells+1]; cell_particles[n] (ascending ids per cell)
int orc_grid_cells(void* hv, int* cell_of, long long* cell_start, int* cell_particles) {
  return guarded([&] {
    with_sim(hv, [&](auto& s) {
      std::copy(s.grid.cell_of.begin(), s.grid.cell_of.end(), cell_of);
      long long k = 0;
      cell_start[0] = 0;
      for (std::size_t c = 0; c < s.grid.cells.size(); ++c) {
        for (int p : s.grid.cells[c]) cell_particles[k++] = p;
        cell_start[c + 1] = k;
      }
    });
  });
}

// block_start[nblocks+1], block_cells[ncells]
int orc_blocks(void* hv, long long* block_start, int* block_cells) {
  return guarded([&] {
    with_sim(hv, [&](auto& s) {
      long long k = 0;
      block_start[0] = 0;
      for (std::size_t b = 0; b < s.blocks.size(); ++b) {
        for (int c : s.blocks[b]) block_cells[k++] = c;
        block_start[b + 1] = k;
      }
    });
  });
}

long long orc_slot_count(void* hv) {
  long long n = 0;
  guarded([&] { with_sim(hv, [&](auto& s) { n = s.nbh.offsets.empty() ? 0 : s.nbh.offsets.back(); }); });
  return n;
}

int orc_get_neighborhood(void* hv, long long* offsets, int* neighbor, double* r0_len, double* e0,
                         double* dwdr0, double* pf) {
  return guarded([&] {
    with_sim(hv, [&](auto& s) {
      constexpr int D = std::remove_reference_t<decltype(s)>::dim;
      const auto& b = s.nbh;
      // any output may be null (not copied)
      if (offsets) std::copy(b.offsets.begin(), b.offsets.end(), offsets);
      if (neighbor) std::copy(b.neighbor.begin(), b.neighbor.end(), neighbor);
      if (r0_len) std::copy(b.r0_len.begin(), b.r0_len.end(), r0_len);
      if (e0)
        for (std::size_t k = 0; k < b.e0.size(); ++k) for (int d = 0; d < D; ++d) e0[k * D + d] = b.e0[k][d];
      if (dwdr0) std::copy(b.dwdr0.begin(), b.dwdr0.end(), dwdr0);
      if (pf) std::copy(b.pair_factor.begin(), b.pair_factor.end(), pf);
    });
  });
}

// Replaces the neighbourhood with a caller-built CSR (hand rigs in the tests).
int orc_set_neighborhood(void* hv, const long long* offsets, const int* neighbor, const double* r0_len,
                         const double* e0, const double* dwdr0, const double* pf) {
  return guarded([&] {
    with_sim(hv, [&](auto& s) {
      constexpr int D = std::remove_reference_t<decltype(s)>::dim;
      const std::size_t n = s.sys.size();
      auto& b = s.nbh;
      b.offsets.assign(offsets, offsets + n + 1);
      const std::size_t total = static_cast<std::size_t>(b.offsets[n]);
      b.neighbor.assign(neighbor, neighbor + total);
      b.r0_len.assign(r0_len, r0_len + total);
      b.dwdr0.assign(dwdr0, dwdr0 + total);
      b.pair_factor.assign(pf, pf + total);
      b.e0.resize(total);
      for (std::size_t k = 0; k < total; ++k) for (int d = 0; d < D; ++d) b.e0[k][d] = e0[k * D + d];
    });
  });
}

// ---- operators (reference operator API)
int orc_correction_matrices(void* hv, int threads) {
  return guarded([&] { with_sim(hv, [&](auto& s) { orc::compute_correction_matrices(s.sys, s.nbh, threads); }); });
}
int orc_deformation_rate(void* hv, int threads) {
  return guarded([&] { with_sim(hv, [&](auto& s) { orc::compute_deformation_rate(s.sys, s.nbh, threads); }); });
}
int orc_update_density(void* hv, int threads) {
  return guarded([&] { with_sim(hv, [&](auto& s) { orc::update_density(s.sys, threads); }); });
}
int orc_momentum_rhs(void* hv, int threads) {
  return guarded([&] { with_sim(hv, [&](auto& s) { orc::compute_momentum_rhs(s.sys, s.nbh, s.mat, s.ext, threads); }); });
}
int orc_verlet_step(void* hv, double dt, int threads) {
  return guarded([&] { with_sim(hv, [&](auto& s) { orc::verlet_step(s.sys, s.nbh, s.mat, s.ext, dt, threads); }); });
}
int orc_apply_constraints(void* hv) {
  return guarded([&] { with_sim(hv, [&](auto& s) { s.sys.apply_constraints(); }); });
}
int orc_stable_dt(void* hv, double h, double* out) {
  return guarded([&] { with_sim(hv, [&](auto& s) { *out = orc::stable_dt(s.sys, s.mat, h); }); });
}
int orc_kinetic_energy(void* hv, double* out) {
  return guarded([&] { with_sim(hv, [&](auto& s) { *out = orc::total_kinetic_energy(s.sys); }); });
}
int orc_check_finite(void* hv, unsigned long long step) {
  return guarded([&] { with_sim(hv, [&](auto& s) { orc::check_finite(s.sys, step); }); });
}
int orc_damping_sweep(void* hv, int scheme, double eta_tilde, double dt, int threads) {
  return guarded([&] {
    with_sim(hv, [&](auto& s) {
      orc::strang_damping_sweep(s.sys, s.nbh, s.grid, s.blocks, static_cast<orc::Scheme>(scheme), eta_tilde, dt, threads);
    });
  });
}
int orc_particle_split_update(void* hv, size_t i, double eta, double dt_half) {
  return guarded([&] { with_sim(hv, [&](auto& s) { orc::particle_split_update(i, s.sys, s.nbh, eta, dt_half); }); });
}
int orc_pairwise_split_update(void* hv, size_t i, long long slot, double eta, double dt_half) {
  return guarded([&] { with_sim(hv, [&](auto& s) { orc::pairwise_split_update(i, slot, s.sys, s.nbh, eta, dt_half); }); });
}
int orc_explicit_damping_accel(void* hv, double eta, double* out, int threads) {
  return guarded([&] {
    with_sim(hv, [&](auto& s) {
      constexpr int D = std::remove_reference_t<decltype(s)>::dim;
      std::vector<orc::Vec<D>> acc;
      orc::explicit_damping_accel(s.sys, s.nbh, eta, acc, threads);
      for (std::size_t i = 0; i < acc.size(); ++i) for (int d = 0; d < D; ++d) out[i * D + d] = acc[i][d];
    });
  });
}

// ---- scalar helpers
int orc_grad_mag(double h, int dim, double r, double* out) {
  return guarded([&] { *out = orc::SmoothingKernel(h, dim).grad_mag(r); });
}
int orc_kernel_value(double h, int dim, double r, double* out) {
  return guarded([&] { *out = orc::SmoothingKernel(h, dim).value(r); });
}
int orc_random_uniforms(unsigned long long seed, size_t n, double* out) {
  return guarded([&] {
    orc::RandomSource rng(seed);
    for (size_t k = 0; k < n; ++k) out[k] = rng.uniform();
  });
}
int orc_random_choice(double eta, double alpha, unsigned long long seed, size_t n, double* out) {
  return guarded([&] {
    orc::RandomSource rng(seed);
    for (size_t k = 0; k < n; ++k) out[k] = orc::random_choice_eta(eta, alpha, rng);
  });
}
int orc_viscous_bounds(double h, double nu_kin, int dim, double* out2) {
  return guarded([&] {
    const auto b = orc::viscous_dt_bounds(h, nu_kin, dim);
    out2[0] = b.explicit_bound;
    out2[1] = b.implicit_bound;
  });
}
int orc_artificial_viscosity(double beta, double rho0, double E, double L, double* out) {
  return guarded([&] { *out = orc::artificial_viscosity(beta, rho0, E, L); });
}
// 3x3 / 2x2 helpers on a single matrix (row-major)
int orc_second_pk(int dim, const double* F, double E, double nu, double rho0, int model, double* out) {
  return guarded([&] {
    const auto mat = orc::material_from_young_poisson(E, nu, rho0, model == 1 ? orc::Model::NeoHookean : orc::Model::LinearKirchhoff);
    auto run = [&](auto tag) {
      constexpr int D = decltype(tag)::value;
      orc::Mat<D> f;
      for (int r = 0; r < D; ++r) for (int c = 0; c < D; ++c) f(r, c) = F[r * D + c];
      const auto S = orc::second_pk<D>(f, mat);
      for (int r = 0; r < D; ++r) for (int c = 0; c < D; ++c) out[r * D + c] = S(r, c);
    };
    if (dim == 2) run(std::integral_constant<int, 2>{});
    else run(std::integral_constant<int, 3>{});
  });
}

// generate_box_lattice (cases.cpp:21-46): returns the count; fills r0 when non-null.
long long orc_box_lattice(int dim, const double* lo, const double* hi, double dp, double* r0_out) {
  long long count = -1;
  guarded([&] {
    auto run = [&](auto tag) {
      constexpr int D = decltype(tag)::value;
      orc::ParticleSystem<D> sys;
      orc::Vec<D> l, u;
      for (int d = 0; d < D; ++d) { l[d] = lo[d]; u[d] = hi[d]; }
      orc::generate_box_lattice<D>(sys, l, u, dp, 1.0);
      count = static_cast<long long>(sys.size());
      if (r0_out) for (std::size_t i = 0; i < sys.size(); ++i) for (int d = 0; d < D; ++d) r0_out[i * D + d] = sys.r0[i][d];
    };
    if (dim == 2) run(std::integral_constant<int, 2>{});
    else run(std::integral_constant<int, 3>{});
  });
  return count;
}

// ---- run loops (the caller side of the path, runner.cpp:341-391, without file output)
// params: [0]=h [1]=eta [2]=alpha [3]=scheme [4]=steps [5]=fixed_dt (<=0: stable_dt)
//         [6]=end_time (<=0: unbounded) [7]=elastic (1: verlet_step each step; 0: damping only)
//         [8]=seed [9]=threads
// out: [0]=steps [1]=damped [2]=t [3]=elastic_s [4]=damping_s [5]=total_s [6]=last_dt
// params[11]: probe particle (-1: none), params[12]: output interval; probe samples (t, u_0..u_2)
// as runner.cpp:328,378-383,393-395 records them: the initial one, one at each output mark, the
// end state if it is later than the last mark.
int orc_run_probed(void* hv, const double* params, double* out, double* samples, long long capacity,
                   long long* nsamples) {
  return guarded([&] {
    with_sim(hv, [&](auto& s) {
      const auto t0 = Clock::now();
      const double h = params[0], eta = params[1], alpha = params[2];
      const auto scheme = static_cast<orc::Scheme>(static_cast<int>(params[3]));
      const long long max_steps = static_cast<long long>(params[4]);
      const double fixed_dt = params[5], end_time = params[6];
      const bool elastic = params[7] != 0.0;
      const auto seed = static_cast<std::uint64_t>(params[8]);
      const int threads = static_cast<int>(params[9]);
      // params[10] != 0: continue the previous run (same RandomSource stream, t and step count;
      // max_steps is cumulative), as the device loop's resume does
      const bool resume = params[10] != 0.0 && s.loop_rng;
      if (!resume) {
        s.loop_rng = std::make_unique<orc::RandomSource>(seed);
        s.loop_t = 0.0;
        s.loop_steps = s.loop_damped = 0;
      }
      orc::RandomSource& rng = *s.loop_rng;
      constexpr int DD = std::remove_reference_t<decltype(s)>::dim;
      const long long probe = params[11] >= 0.0 ? static_cast<long long>(params[11]) : -1;
      const double interval = params[12];
      long long ns = 0;
      auto record = [&](double tt) {
        if (probe < 0 || !samples || ns >= capacity) return;
        double* o = samples + 4 * ns++;
        o[0] = tt;
        o[1] = o[2] = o[3] = 0.0;
        for (int d = 0; d < DD; ++d) o[1 + d] = s.sys.r[static_cast<std::size_t>(probe)][d] - s.sys.r0[static_cast<std::size_t>(probe)][d];
      };
      if (!resume) record(0.0);
      double next_mark = interval > 0.0 ? interval : 0.0;
      const bool damping_active = eta > 0.0;
      orc::ViscousBounds vb{};
      if (damping_active) vb = orc::viscous_dt_bounds(h, eta / (alpha * s.mat.rho0), std::remove_reference_t<decltype(s)>::dim);
      double t = s.loop_t, el = 0.0, dm = 0.0, last_dt = 0.0;
      long long steps = s.loop_steps, damped = s.loop_damped;
      std::vector<orc::Vec<std::remove_reference_t<decltype(s)>::dim>> visc;
      // a failing step leaves the completed-step count and t behind (orc_last_run), as
      // tlsph_dev_last_run_steps does for the device loop
      struct Completed {
        decltype(s)& sim;
        long long& steps;
        double& t;
        bool armed = true;
        ~Completed() {
          if (armed) {
            sim.loop_steps = steps;
            sim.loop_t = t;
          }
        }
      };
      Completed completed{s, steps, t};
      while ((end_time <= 0.0 || t < end_time) && steps < max_steps) {
        double dt = fixed_dt > 0.0 ? fixed_dt : orc::stable_dt(s.sys, s.mat, h);
        if (damping_active && fixed_dt <= 0.0) {
          if (scheme == orc::Scheme::Explicit) dt = std::min(dt, vb.explicit_bound);
          else if (scheme == orc::Scheme::ParticleSplit) dt = std::min(dt, vb.implicit_bound);
        }
        if (end_time > 0.0) dt = std::min(dt, end_time - t);
        last_dt = dt;
        if (elastic) {
          const auto te = Clock::now();
          orc::verlet_step(s.sys, s.nbh, s.mat, s.ext, dt, threads);
          el += since(te);
        }
        if (damping_active) {
          const auto td = Clock::now();
          const double eta_tilde = orc::random_choice_eta(eta, alpha, rng);
          if (eta_tilde > 0.0) {
            ++damped;
            if (scheme == orc::Scheme::Explicit) {
              orc::explicit_damping_accel(s.sys, s.nbh, eta_tilde, visc, threads);
              for (std::size_t i = 0; i < s.sys.size(); ++i)
                for (int d = 0; d < std::remove_reference_t<decltype(s)>::dim; ++d) s.sys.v[i][d] = s.sys.v[i][d] + dt * visc[i][d];
            } else {
              orc::strang_damping_sweep(s.sys, s.nbh, s.grid, s.blocks, scheme, eta_tilde, dt, threads);
            }
            s.sys.apply_constraints();
          }
          dm += since(td);
        }
        t += dt;
        ++steps;
        orc::check_finite(s.sys, static_cast<std::uint64_t>(steps));
        if (probe >= 0 && interval > 0.0 && t >= next_mark - 1e-12 * end_time) {
          record(t);
          while (next_mark <= t + 1e-12 * end_time) next_mark += interval;
        }
      }
      if (probe >= 0 && (ns == 0 || samples[4 * (ns - 1)] < t)) record(t);
      if (nsamples) *nsamples = ns;
      completed.armed = false;
      s.loop_t = t;
      s.loop_steps = steps;
      s.loop_damped = damped;
      out[0] = static_cast<double>(steps);
      out[1] = static_cast<double>(damped);
      out[2] = t;
      out[3] = el;
      out[4] = dm;
      out[5] = since(t0);
      out[6] = last_dt;
    });
  });
}

int orc_run(void* hv, const double* params, double* out) {
  double p[13];
  for (int k = 0; k < 11; ++k) p[k] = params[k];
  p[11] = -1.0;
  p[12] = 0.0;
  return orc_run_probed(hv, p, out, nullptr, 0, nullptr);
}

// Completed steps and t of the last run, also when it stopped on an error.
int orc_last_run(void* hv, double* out) {
  return guarded([&] {
    with_sim(hv, [&](auto& s) {
      out[0] = static_cast<double>(s.loop_steps);
      out[1] = s.loop_t;
    });
  });
}

// ExternalAccel's contact plane (forces.hpp:13-24); stiffness <= 0 removes it.
int orc_set_contact(void* hv, const double* point, const double* normal, double stiffness) {
  return guarded([&] {
    with_sim(hv, [&](auto& s) {
      constexpr int DD = std::remove_reference_t<decltype(s)>::dim;
      s.ext.contact = stiffness > 0.0;
      s.ext.cp_k = stiffness;
      for (int d = 0; d < DD; ++d) {
        s.ext.cp_point[d] = point[d];
        s.ext.cp_normal[d] = normal[d];
      }
    });
  });
}

// Initialisation the runner performs before the loop (runner.cpp:306-312):
// B0, constraints, initial momentum RHS and deformation rate.
int orc_prepare(void* hv, int threads) {
  return guarded([&] {
    with_sim(hv, [&](auto& s) {
      orc::compute_correction_matrices(s.sys, s.nbh, threads);
      s.sys.apply_constraints();
      orc::compute_momentum_rhs(s.sys, s.nbh, s.mat, s.ext, threads);
      orc::compute_deformation_rate(s.sys, s.nbh, threads);
    });
  });
}

}  // extern "C"
