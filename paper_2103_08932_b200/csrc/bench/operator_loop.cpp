// End-to-end measurement through the reference's C++ operator API (bench.py's `e2e` legs).
//
// A reference caller drops this library in and keeps calling the operators it already calls, on
// its own host ParticleSystem<3> (std::vector storage, pageable): the loop below is the one of
// proj/src/tlsph/runner.cpp:341-391 (stable_dt -> verlet_step -> random_choice_eta ->
// strang_damping_sweep -> apply_constraints -> check_finite), written against include/tlsph/*.hpp
// only. Every operator moves the particle fields it reads host -> device and the ones it writes
// device -> host, inside the timed region; the neighbourhood stays resident on the device
// (csrc/host/resident.hpp).
//
//   tlsph-operator-loop sweep <steps> <warmup> [fast|ordered] [pinned|pageable]   cfg2: strang_damping_sweep<3>
//   tlsph-operator-loop loop  <steps> <warmup> [fast|ordered] [pinned|pageable]   cfg4: the runner loop
// pinned (default): the caller page-locks its ParticleSystem once (tlsph::pin_host_memory) before
// the loop, as a GPU-aware caller does; pageable: plain std::vector storage (staging ring).
//
// Inputs follow BASELINE.md §3 (generate_box_lattice, RandomSource streams). Prints one JSON line.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <span>
#include <string>

#include "tlsph/cases.hpp"
#include "tlsph/damping.hpp"
#include "tlsph/device.hpp"
#include "tlsph/errors.hpp"
#include "tlsph/integrator.hpp"
#include "tlsph/material.hpp"
#include "tlsph/neighbors.hpp"
#include "tlsph/tlsph_dev.h"

using namespace tlsph;
using Clock = std::chrono::steady_clock;

namespace {

constexpr double kRho0 = 1000.0, kE = 2.0e6, kNu = 0.3, kGravity = 9.81;

bool g_pinned = true;  // the caller page-locks its ParticleSystem (tlsph/device.hpp); "pageable" arg: off

double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

struct Bytes {
  std::uint64_t h2d = 0, d2h = 0;
  static Bytes now() {
    Bytes b;
    tlsph_dev_transfer_bytes(&b.h2d, &b.d2h);
    return b;
  }
};

// runner.cpp:233-247 (the caller's own per-step check)
void check_finite(const ParticleSystem<3>& s, std::uint64_t step) {
  double total = 0.0;
  for (std::size_t i = 0; i < s.size(); ++i) total += s.v[i].squaredNorm() + s.r[i].squaredNorm();
  if (std::isfinite(total)) return;
  for (std::size_t i = 0; i < s.size(); ++i)
    if (!s.v[i].allFinite() || !s.r[i].allFinite())
      throw Error(ErrorKind::NumericalFailure,
                  "NaN detected at step " + std::to_string(step) + ", particle " + std::to_string(i));
}

int sweep_bench(int steps, int warmup) {
  // cfg2: 64^3 on [0,1]^3, v ~ N(0,1) by Box-Muller on RandomSource(1), alpha 1, dt = 0.6 h / c
  const double dp = 1.0 / 64, h = 1.3 * dp;
  ParticleSystem<3> sys;
  generate_box_lattice<3>(sys, Vec3(0, 0, 0), Vec3(1, 1, 1), dp, kRho0);
  const std::size_t n = sys.size();
  RandomSource rng(1);
  std::vector<double> z(n * 3);
  for (std::size_t k = 0; k < z.size(); k += 2) {
    const double u1 = rng.uniform(), u2 = rng.uniform();
    const double rho = std::sqrt(-2.0 * std::log(1.0 - u1));
    z[k] = rho * std::cos(2.0 * M_PI * u2);
    if (k + 1 < z.size()) z[k + 1] = rho * std::sin(2.0 * M_PI * u2);
  }
  for (std::size_t i = 0; i < n; ++i) sys.v[i] = Vec3(z[3 * i], z[3 * i + 1], z[3 * i + 2]);
  const Material mat = material_from_young_poisson(kE, kNu, kRho0, ConstitutiveModel::NeoHookean);
  const double eta = 0.2 * kRho0 * mat.c * h, dt = 0.6 * h / mat.c;

  const auto t_init = Clock::now();
  const auto grid = build_cell_grid<3>(std::span<const Vec3>(sys.r0), 2.0 * h);
  const auto blocks = block_decompose<3>(grid);
  const SmoothingKernel kernel(h, 3);
  const auto nbh = build_reference_neighborhoods<3>(std::span<const Vec3>(sys.r0), std::span<const double>(sys.V0),
                                                    kernel, grid);
  const double init_s = since(t_init);
  if (g_pinned) pin_host_memory<3>(sys);
  for (int k = 0; k < warmup; ++k)
    strang_damping_sweep<3>(sys, nbh, grid, blocks, DampingScheme::ParticleSplit, eta, dt, 1);
  const Bytes b0 = Bytes::now();
  const auto t0 = Clock::now();
  for (int k = 0; k < steps; ++k)
    strang_damping_sweep<3>(sys, nbh, grid, blocks, DampingScheme::ParticleSplit, eta, dt, 1);
  const double secs = since(t0);
  const Bytes b1 = Bytes::now();
  if (g_pinned) unpin_host_memory<3>(sys);
  std::int64_t s_free = nbh.offsets.back();
  const double dpu = 2.0 * static_cast<double>(s_free) * steps;
  std::printf("{\"workload\": \"cfg2\", \"api\": \"tlsph::strang_damping_sweep<3> on a host ParticleSystem<3>\", "
              "\"particles\": %zu, \"slots\": %lld, \"steps\": %d, \"warmup\": %d, \"seconds\": %.9g, "
              "\"value\": %.9g, \"unit\": \"DPU/s\", \"h2d_bytes_per_step\": %llu, \"d2h_bytes_per_step\": %llu, "
              "\"init_seconds\": %.6g, \"var_v\": %.17g, \"host_memory\": \"%s\"}\n",
              n, static_cast<long long>(s_free), steps, warmup, secs, dpu / secs,
              static_cast<unsigned long long>((b1.h2d - b0.h2d) / std::max(steps, 1)),
              static_cast<unsigned long long>((b1.d2h - b0.d2h) / std::max(steps, 1)), init_s,
              [&] {
                double m = 0, q = 0;
                for (auto& x : sys.v)
                  for (int d = 0; d < 3; ++d) m += x[d];
                m /= 3.0 * n;
                for (auto& x : sys.v)
                  for (int d = 0; d < 3; ++d) q += (x[d] - m) * (x[d] - m);
                return q / (3.0 * n);
              }(),
              g_pinned ? "pinned" : "pageable");
  return 0;
}

int loop_bench(int steps, int warmup) {
  // cfg4: [0,1]x[0,1]x[0,0.5] at dp 0.004, r0 jittered by (2u-1) 0.4 dp from RandomSource(3), v
  // from the same stream; 5-layer clamp; gravity; alpha 0.1, damping seed 0
  const double dp = 0.004, h = 1.3 * dp;
  ParticleSystem<3> sys;
  generate_box_lattice<3>(sys, Vec3(0, 0, 0), Vec3(1.0, 1.0, 0.5), dp, kRho0);
  const std::size_t n = sys.size();
  RandomSource init(3);
  for (std::size_t i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) sys.r0[i][d] = sys.r0[i][d] + (2.0 * init.uniform() - 1.0) * (0.4 * dp);
  for (std::size_t i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) sys.v[i][d] = -0.01 + 0.02 * init.uniform();
  for (std::size_t i = 0; i < n; ++i) {
    sys.r[i] = sys.r0[i];
    sys.constrained[i] = sys.r0[i][0] < 5 * dp ? 1 : 0;
  }
  ExternalAccel<3> ext;
  ext.body.assign(n, Vec3(0.0, -kGravity, 0.0));
  const Material mat = material_from_young_poisson(kE, kNu, kRho0, ConstitutiveModel::NeoHookean);
  DampingConfig damping;
  damping.eta = 0.2 * kRho0 * mat.c * h;
  damping.alpha = 0.1;
  damping.seed = 0;

  // runner.cpp:299-312
  const auto t_init = Clock::now();
  const auto grid = build_cell_grid<3>(std::span<const Vec3>(sys.r0), 2.0 * h);
  const auto blocks = block_decompose<3>(grid);
  const SmoothingKernel kernel(h, 3);
  const auto nbh = build_reference_neighborhoods<3>(std::span<const Vec3>(sys.r0), std::span<const double>(sys.V0),
                                                    kernel, grid);
  compute_correction_matrices<3>(sys, nbh, 1);
  sys.apply_constraints();
  compute_momentum_rhs<3>(sys, nbh, mat, ext, 1);
  compute_deformation_rate<3>(sys, nbh, 1);
  const double init_s = since(t_init);
  RandomSource rng(damping.seed);
  const ViscousBounds viscous = viscous_dt_bounds(h, damping.nu_kin_applied(kRho0), 3);
  if (g_pinned) pin_host_memory<3>(sys, &ext.body);

  std::uint64_t step = 0, damped = 0, damped_timed = 0;
  double t = 0.0;
  double caller_s = 0.0;  // the caller's own serial host code inside the loop (constraints, finite check)
  auto one_step = [&] {  // runner.cpp:341-377
    StepSizes sizes = stable_dt<3>(sys, mat, h);
    sizes.dt = std::min(sizes.dt, viscous.implicit_bound);
    const double dt = sizes.dt;
    verlet_step<3>(sys, nbh, mat, ext, dt, 1);
    const double eta_tilde = random_choice_eta(damping.eta, damping.alpha, rng);
    bool was_damped = false;
    if (eta_tilde > 0.0) {
      ++damped;
      was_damped = true;
      strang_damping_sweep<3>(sys, nbh, grid, blocks, DampingScheme::ParticleSplit, eta_tilde, dt, 1);
      const auto tc = Clock::now();
      sys.apply_constraints();
      caller_s += since(tc);
    }
    t += dt;
    ++step;
    const auto tc = Clock::now();
    check_finite(sys, step);
    caller_s += since(tc);
    return was_damped;
  };
  for (int k = 0; k < warmup; ++k) one_step();
  const Bytes b0 = Bytes::now();
  caller_s = 0.0;
  const auto t0 = Clock::now();
  for (int k = 0; k < steps; ++k) damped_timed += one_step() ? 1 : 0;
  const double secs = since(t0);
  const double caller_timed = caller_s;
  const Bytes b1 = Bytes::now();
  if (g_pinned) unpin_host_memory<3>(sys, &ext.body);
  double disp = 0.0;
  for (std::size_t i = 0; i < n; ++i) disp += (sys.r[i] - sys.r0[i]).squaredNorm();
  std::printf("{\"workload\": \"cfg4\", \"api\": \"runner.cpp:341-391 loop over tlsph::stable_dt / verlet_step / "
              "strang_damping_sweep<3> on a host ParticleSystem<3>\", \"particles\": %zu, \"slots\": %lld, "
              "\"steps\": %d, \"warmup\": %d, \"damped_steps\": %llu, \"seconds\": %.9g, \"value\": %.9g, "
              "\"unit\": \"PS/s\", \"h2d_bytes_per_step\": %llu, \"d2h_bytes_per_step\": %llu, "
              "\"init_seconds\": %.6g, \"t\": %.17g, \"displacement_l2\": %.17g, \"host_memory\": \"%s\", "
              "\"caller_host_seconds\": %.6g}\n",
              n, static_cast<long long>(nbh.offsets.back()), steps, warmup,
              static_cast<unsigned long long>(damped_timed), secs, static_cast<double>(n) * steps / secs,
              static_cast<unsigned long long>((b1.h2d - b0.h2d) / std::max(steps, 1)),
              static_cast<unsigned long long>((b1.d2h - b0.d2h) / std::max(steps, 1)), init_s, t, std::sqrt(disp),
              g_pinned ? "pinned" : "pageable", caller_timed);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s sweep|loop <steps> <warmup> [fast|ordered]\n", argv[0]);
    return 2;
  }
  const std::string what = argv[1];
  const int steps = std::atoi(argv[2]), warmup = std::atoi(argv[3]);
  const std::string mode = argc > 4 ? argv[4] : "fast";
  g_pinned = !(argc > 5 && std::string(argv[5]) == "pageable");
  set_operator_reduction(mode == "ordered" ? Reduction::Ordered : Reduction::Fast);
  try {
    if (what == "sweep") return sweep_bench(steps, warmup);
    if (what == "loop") return loop_bench(steps, warmup);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "operator_loop: %s\n", e.what());
    return 1;
  }
  std::fprintf(stderr, "unknown workload %s\n", what.c_str());
  return 2;
}
