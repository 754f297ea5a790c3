// Ports of the reference's doctest suites (proj/tests/test_{neighbors,damping,
// integrator,runner}.cpp) against this build's C++ operator API: the same
// calls, the same known answers, but every operator runs on the B200 through
// the C ABI of tlsph_dev.h.
#include <algorithm>
#include <cstdint>
#include <filesystem>
#include <fstream>
#include <random>
#include <set>
#include <sstream>

#include "harness.hpp"
#include "tlsph/damping.hpp"
#include "tlsph/errors.hpp"
#include "tlsph/integrator.hpp"
#include "tlsph/neighbors.hpp"
#include "tlsph/runner.hpp"

using namespace tlsph;

namespace {

template <int D>
struct Fixture {
  ParticleSystem<D> system;
  CellGrid<D> grid;
  BlockDecomposition<D> blocks;
  ReferenceNeighborhood<D> nbh;
  double h = 0.0;
};

// test_support.hpp:27-60
template <int D>
Fixture<D> lattice_fixture(const std::array<int, D>& counts, double dp, double rho0) {
  Fixture<D> fx;
  std::array<int, D> idx{};
  for (;;) {
    Vec<D> p;
    for (int d = 0; d < D; ++d) p[d] = (idx[d] + 0.5) * dp;
    fx.system.add_particle(p, std::pow(dp, D), rho0);
    int d = 0;
    while (d < D && ++idx[d] >= counts[d]) idx[d++] = 0;
    if (d == D) break;
  }
  fx.h = 1.3 * dp;
  const SmoothingKernel kernel(fx.h, D);
  fx.grid = build_cell_grid<D>(std::span<const Vec<D>>(fx.system.r0), kernel.support_radius());
  fx.blocks = block_decompose<D>(fx.grid);
  fx.nbh = build_reference_neighborhoods<D>(std::span<const Vec<D>>(fx.system.r0),
                                            std::span<const double>(fx.system.V0), kernel, fx.grid);
  return fx;
}

template <int D>
void randomize(ParticleSystem<D>& s, double scale, std::mt19937& gen) {
  std::uniform_real_distribution<double> dist(-scale, scale);
  for (auto& v : s.v)
    for (int d = 0; d < D; ++d) v[d] = dist(gen);
}

template <int D>
Vec<D> momentum(const ParticleSystem<D>& s) {
  Vec<D> p = Vec<D>::Zero();
  for (std::size_t i = 0; i < s.size(); ++i) p += s.m[i] * s.v[i];
  return p;
}

}  // namespace

// ---------------------------------------------------------------- neighbours
TEST_CASE("block membership matches the published 9x6 example") {  // test_neighbors.cpp:95-113
  std::vector<Vec2> pts;
  for (int iy = 0; iy < 6; ++iy)
    for (int ix = 0; ix < 9; ++ix) pts.push_back(Vec2(ix + 0.5, iy + 0.5));
  const auto grid = build_cell_grid<2>(std::span<const Vec2>(pts), 1.0);
  REQUIRE(grid.dims[0] == 9 && grid.dims[1] == 6);
  const auto blocks = block_decompose<2>(grid);
  CHECK((blocks.blocks[0] == std::vector<int>{0, 3, 6, 27, 30, 33}));
  CHECK((blocks.blocks[8] == std::vector<int>{20, 23, 26, 47, 50, 53}));
}

TEST_CASE("empty particle set and coincident particles are rejected") {  // :50-53, :238-245
  std::vector<Vec2> none;
  CHECK_THROWS(build_cell_grid<2>(std::span<const Vec2>(none), 0.5));
  SmoothingKernel kernel(0.1, 2);
  std::vector<Vec2> pts{Vec2(0.4, 0.4), Vec2(0.4, 0.4)};
  std::vector<double> vol(2, 1.0);
  const auto grid = build_cell_grid<2>(std::span<const Vec2>(pts), kernel.support_radius());
  bool degenerate = false;
  try {
    build_reference_neighborhoods<2>(std::span<const Vec2>(pts), std::span<const double>(vol), kernel, grid);
  } catch (const Error& e) {
    degenerate = e.kind() == ErrorKind::DegenerateGeometry;
  }
  CHECK(degenerate);
}

TEST_CASE("stencil candidates cover all brute-force pairs; rows ascending, symmetric") {  // :66-93, :198-224
  std::mt19937 gen(5);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  std::vector<Vec3> pts(300);
  for (auto& p : pts) p = Vec3(u(gen), u(gen), u(gen));
  SmoothingKernel kernel(0.06, 3);
  std::vector<double> vol(pts.size(), 1e-6);
  const auto grid = build_cell_grid<3>(std::span<const Vec3>(pts), kernel.support_radius());
  const auto nbh = build_reference_neighborhoods<3>(std::span<const Vec3>(pts), std::span<const double>(vol), kernel, grid);
  std::set<std::pair<int, int>> exact, got;
  for (std::size_t i = 0; i < pts.size(); ++i)
    for (std::size_t j = 0; j < pts.size(); ++j)
      if (i != j && (pts[i] - pts[j]).norm() < 0.12) exact.emplace(int(i), int(j));
  for (std::size_t i = 0; i < pts.size(); ++i) {
    CHECK(std::is_sorted(nbh.neighbor.begin() + nbh.begin(i), nbh.neighbor.begin() + nbh.end(i)));
    for (auto s = nbh.begin(i); s < nbh.end(i); ++s) {
      got.emplace(int(i), nbh.neighbor[s]);
      CHECK(nbh.pair_factor[s] <= 0.0);
    }
  }
  CHECK(got == exact);
}

TEST_CASE("lattice interior neighbor count is 20") {  // :247-276
  auto fx = lattice_fixture<2>({12, 12}, 0.01, 1.0);
  std::size_t c = 0;
  double best = 1e30;
  for (std::size_t i = 0; i < fx.system.size(); ++i) {
    const double d = (fx.system.r0[i] - Vec2(0.06, 0.06)).norm();
    if (d < best) {
      best = d;
      c = i;
    }
  }
  CHECK(fx.nbh.count(c) == 20);
}

TEST_CASE("reverse pass visits blocks and cells in mirrored order") {  // :303-326
  std::vector<Vec2> pts;
  for (int iy = 0; iy < 5; ++iy)
    for (int ix = 0; ix < 7; ++ix) pts.push_back(Vec2(ix + 0.5, iy + 0.5));
  const auto grid = build_cell_grid<2>(std::span<const Vec2>(pts), 1.0);
  const auto blocks = block_decompose<2>(grid);
  std::vector<int> fwd, full;
  block_sweep<2>(blocks, [&](int c, SweepDirection) { fwd.push_back(c); }, SweepSchedule::Forward, 1);
  block_sweep<2>(blocks, [&](int c, SweepDirection) { full.push_back(c); }, SweepSchedule::ForwardThenReverse, 1);
  REQUIRE(full.size() == 2 * fwd.size());
  CHECK((std::vector<int>(full.begin() + fwd.size(), full.end()) == std::vector<int>(fwd.rbegin(), fwd.rend())));
}

// ---------------------------------------------------------------- damping
TEST_CASE("particle split single-neighbor update matches the scalar re-derivation") {  // test_damping.cpp:147-170
  ParticleSystem<3> s;
  s.add_particle(Vec3::Zero(), 1.0, 1.0);
  s.add_particle(Vec3(1.0, 0.0, 0.0), 1.0, 1.0);
  ReferenceNeighborhood<3> nbh;
  nbh.offsets = {0, 1, 2};
  nbh.neighbor = {1, 0};
  nbh.r0_len = {1.0, 1.0};
  nbh.e0 = {Vec3(1.0, 0.0, 0.0), Vec3(-1.0, 0.0, 0.0)};
  nbh.dwdr0 = {-0.05, -0.05};
  nbh.pair_factor = {-0.1, -0.1};
  s.v[0] = Vec3(1.0, 0.0, 0.0);
  particle_split_update(std::size_t{0}, s, nbh, 1.0, 1.0);
  const double B = -0.1, diag = B - 1.0, k = (-B) / (diag * diag + B * B);
  const double vin = 1.0 + diag * k, vjn = 0.0 - B * (vin - (0.0 - B * k)) / 1.0;
  CHECK(th::approx(s.v[0][0], vin, 1e-14));
  CHECK(th::approx(s.v[1][0], vjn, 1e-14));
  CHECK(th::approx(s.v[0][0] + s.v[1][0], 1.0, 1e-14));
}

TEST_CASE("pairwise update solves the 2x2 implicit system exactly") {  // :219-268
  std::mt19937 gen(19);
  std::uniform_real_distribution<double> mass(0.1, 10.0), factor(-5.0, -1e-4), vel(-2.0, 2.0);
  for (int trial = 0; trial < 50; ++trial) {
    const double mi = mass(gen), mj = mass(gen), B = factor(gen);
    ParticleSystem<3> s;
    s.add_particle(Vec3::Zero(), 1.0, mi);
    s.add_particle(Vec3(1.0, 0.0, 0.0), 1.0, mj);
    ReferenceNeighborhood<3> nbh;
    nbh.offsets = {0, 1, 2};
    nbh.neighbor = {1, 0};
    nbh.r0_len = {1.0, 1.0};
    nbh.e0 = {Vec3(1.0, 0.0, 0.0), Vec3(-1.0, 0.0, 0.0)};
    nbh.dwdr0 = {B / 2, B / 2};
    nbh.pair_factor = {B, B};
    for (int d = 0; d < 3; ++d) {
      s.v[0][d] = vel(gen);
      s.v[1][d] = vel(gen);
    }
    const Vec3 vi = s.v[0], vj = s.v[1], vij = vi - vj;
    pairwise_split_update(std::size_t{0}, std::int64_t{0}, s, nbh, 1.0, 1.0);
    for (int d = 0; d < 3; ++d) {
      const double x = vij[d], a11 = mi - B, a22 = mj - B, det = a11 * a22 - B * B;
      CHECK(th::approx(s.v[0][d] - vi[d], (B * x * a22 - B * (-B * x)) / det, 1e-12));
      CHECK(th::approx(s.v[1][d] - vj[d], (a11 * (-B * x) - B * x * B) / det, 1e-12));
    }
  }
}

TEST_CASE("full sweeps conserve momentum; zero eta is a no-op; uniform field invariant") {  // :295-346
  for (auto scheme : {DampingScheme::ParticleSplit, DampingScheme::PairwiseSplit}) {
    auto fx = lattice_fixture<2>({9, 9}, 0.01, 1000.0);
    std::mt19937 gen(29);
    randomize<2>(fx.system, 1.0, gen);
    const Vec2 before = momentum(fx.system);
    double scale = 0.0;
    for (std::size_t i = 0; i < fx.system.size(); ++i) scale += fx.system.m[i] * fx.system.v[i].norm();
    strang_damping_sweep(fx.system, fx.nbh, fx.grid, fx.blocks, scheme, 160.0, 1e-4, 1);
    CHECK((momentum(fx.system) - before).norm() <= 1e-10 * scale);
  }
  auto fx = lattice_fixture<2>({5, 5}, 0.01, 1000.0);
  std::mt19937 gen(37);
  randomize<2>(fx.system, 1.0, gen);
  const auto v0 = fx.system.v;
  strang_damping_sweep(fx.system, fx.nbh, fx.grid, fx.blocks, DampingScheme::ParticleSplit, 0.0, 1e-4, 1);
  CHECK(fx.system.v == v0);
  auto f3 = lattice_fixture<3>({4, 4, 4}, 0.01, 1265.0);
  for (auto& v : f3.system.v) v = Vec3(0.2, -0.5, 0.9);
  strang_damping_sweep(f3.system, f3.nbh, f3.grid, f3.blocks, DampingScheme::ParticleSplit, 160.0, 1e-4, 1);
  for (const auto& v : f3.system.v) CHECK((v - Vec3(0.2, -0.5, 0.9)).norm() <= 1e-15);
}

TEST_CASE("sweep order matches a scripted 1D-chain application") {  // :348-436
  const double dp = 0.01;
  ParticleSystem<2> system;
  for (int i = 0; i < 5; ++i) system.add_particle(Vec2((i + 0.5) * dp, 0.5 * dp), dp * dp, 1000.0);
  const SmoothingKernel kernel(1.3 * dp, 2);
  const auto grid = build_cell_grid<2>(std::span<const Vec2>(system.r0), kernel.support_radius());
  REQUIRE(grid.cell_count() == 2);
  REQUIRE((grid.cells[0] == std::vector<int>{0, 1, 2}));
  const auto blocks = block_decompose<2>(grid);
  const auto nbh = build_reference_neighborhoods<2>(std::span<const Vec2>(system.r0),
                                                    std::span<const double>(system.V0), kernel, grid);
  std::mt19937 gen(41);
  std::uniform_real_distribution<double> vel(-1.0, 1.0);
  for (auto& v : system.v) v = Vec2(vel(gen), vel(gen));
  const double eta = 100.0, dt = 2e-4;
  ParticleSystem<2> swept = system, replay = system;
  strang_damping_sweep(swept, nbh, grid, blocks, DampingScheme::ParticleSplit, eta, dt, 1);
  auto apply = [&](std::size_t i, double tau) {
    Vec2 res = Vec2::Zero();
    double sb = 0.0, sb2 = 0.0;
    for (auto s = nbh.begin(i); s < nbh.end(i); ++s) {
      const auto j = static_cast<std::size_t>(nbh.neighbor[s]);
      const double b = eta * nbh.pair_factor[s] * tau;
      res -= b * (replay.v[i] - replay.v[j]);
      sb += b;
      sb2 += b * b;
    }
    const double diag = sb - replay.m[i];
    const Vec2 k = res / (diag * diag + sb2);
    const Vec2 vin = replay.v[i] + diag * k;
    for (auto s = nbh.begin(i); s < nbh.end(i); ++s) {
      const auto j = static_cast<std::size_t>(nbh.neighbor[s]);
      const double b = eta * nbh.pair_factor[s] * tau;
      const Vec2 pred = replay.v[j] - b * k;
      replay.v[j] -= (b / replay.m[j]) * (vin - pred);
    }
    replay.v[i] = vin;
  };
  for (int idx : {0, 1, 2, 3, 4, 4, 3, 2, 1, 0}) apply(static_cast<std::size_t>(idx), 0.5 * dt);
  for (std::size_t i = 0; i < replay.size(); ++i)
    CHECK((swept.v[i] - replay.v[i]).norm() <= 1e-14 * (1.0 + replay.v[i].norm()));
}

TEST_CASE("random choice: application fraction and mean are unbiased") {  // :72-90
  RandomSource rng(42);
  int applied = 0;
  double sum = 0.0;
  for (int k = 0; k < 100000; ++k) {
    const double v = random_choice_eta(32.0, 0.2, rng);
    applied += v > 0.0;
    sum += v;
  }
  CHECK(std::abs(applied / 100000.0 - 0.2) <= 0.01);
  CHECK(std::abs(sum / 100000.0 - 32.0) <= 0.02 * 32.0);
}

// ---------------------------------------------------------------- integrator
TEST_CASE("correction matrix restores linear completeness everywhere") {  // test_integrator.cpp:15-30
  auto fx = lattice_fixture<2>({10, 10}, 0.01, 1000.0);
  compute_correction_matrices(fx.system, fx.nbh, 1);
  Mat2 L;
  L << 0.3, -1.2, 0.7, 0.4;
  for (std::size_t i = 0; i < fx.system.size(); ++i) fx.system.v[i] = L * fx.system.r0[i];
  compute_deformation_rate(fx.system, fx.nbh, 1);
  double Ln = 0.0;
  for (int k = 0; k < 4; ++k) Ln += L.data()[k] * L.data()[k];
  for (const auto& r : fx.system.dFdt) {
    double e = 0.0;
    for (int k = 0; k < 4; ++k) e += (r.data()[k] - L.data()[k]) * (r.data()[k] - L.data()[k]);
    CHECK(std::sqrt(e) <= 1e-10 * std::sqrt(Ln));
  }
}

TEST_CASE("density follows rho0 / det(F); inverted element rejected") {  // :108-133
  auto fx = lattice_fixture<3>({3, 3, 3}, 0.01, 1265.0);
  fx.system.F[0] = Vec3(2.0, 1.0, 1.0).asDiagonal();
  update_density(fx.system, 1);
  CHECK(th::approx(fx.system.rho[0], 632.5, 1e-14));
  fx.system.F[2] = -Mat3::Identity();
  bool inverted = false;
  try {
    update_density(fx.system, 1);
  } catch (const Error& e) {
    inverted = e.kind() == ErrorKind::InvertedElement &&
               std::string(e.what()) == "inverted element: det(F) <= 0 for particle 2";
  }
  CHECK(inverted);
}

TEST_CASE("momentum RHS: stress-free body feels only the body force; momentum conserved") {  // :135-175
  auto fx = lattice_fixture<3>({5, 4, 3}, 0.01, 1265.0);
  compute_correction_matrices(fx.system, fx.nbh, 1);
  const Material mat = material_from_young_poisson(5e4, 0.45, 1265.0, ConstitutiveModel::NeoHookean);
  ExternalAccel<3> gravity;
  gravity.body.assign(fx.system.size(), Vec3(0.0, -9.8, 0.0));
  compute_momentum_rhs(fx.system, fx.nbh, mat, gravity, 1);
  for (const auto& a : fx.system.a) CHECK((a - Vec3(0.0, -9.8, 0.0)).norm() <= 1e-12 * 9.8);
  std::mt19937 gen(7);
  std::uniform_real_distribution<double> entry(-0.02, 0.02);
  for (auto& F : fx.system.F)
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) F(r, c) += entry(gen);
  ExternalAccel<3> none;
  compute_momentum_rhs(fx.system, fx.nbh, mat, none, 1);
  Vec3 total = Vec3::Zero();
  double scale = 0.0;
  for (std::size_t i = 0; i < fx.system.size(); ++i) {
    total += fx.system.m[i] * fx.system.a[i];
    scale += fx.system.m[i] * fx.system.a[i].norm();
  }
  CHECK(total.norm() <= 1e-10 * scale);
}

TEST_CASE("verlet step is exact for a constant body force") {  // :205-224
  ParticleSystem<3> s;
  s.add_particle(Vec3::Zero(), 1.0, 1.0);
  s.v[0] = Vec3(0.2, 0.1, 0.0);
  ReferenceNeighborhood<3> nbh;
  nbh.offsets = {0, 0};
  const Material mat = material_from_young_poisson(1e5, 0.3, 1.0, ConstitutiveModel::LinearKirchhoff);
  ExternalAccel<3> gravity;
  gravity.body.assign(1, Vec3(0.0, -9.8, 0.0));
  const double dt = 1e-3;
  const Vec3 r0 = s.r[0], v0 = s.v[0], g(0.0, -9.8, 0.0);
  verlet_step(s, nbh, mat, gravity, dt, 1);
  CHECK((s.v[0] - (v0 + dt * g)).norm() <= 1e-15);
  CHECK((s.r[0] - (r0 + dt * v0 + 0.5 * dt * dt * g)).norm() <= 1e-15);
}

TEST_CASE("stable step size reproduces the coarse-cantilever arithmetic") {  // :273-294
  auto fx = lattice_fixture<3>({3, 3, 3}, 0.04 / 6.0, 1265.0);
  const Material mat = material_from_young_poisson(5e4, 0.45, 1265.0, ConstitutiveModel::NeoHookean);
  const double h = 1.3 * 0.04 / 6.0;
  for (auto& a : fx.system.a) a = Vec3(0.0, -9.8, 0.0);
  CHECK(th::approx(stable_dt(fx.system, mat, h).dt_acoustic, 4.53e-4, 2e-3));
  for (auto& a : fx.system.a) a.setZero();
  CHECK(th::approx(stable_dt(fx.system, mat, h).dt_acoustic, 0.6 * h / mat.c, 1e-12));
}

// ---------------------------------------------------------------- runner
namespace {
std::string read_file(const std::string& p) {
  std::ifstream in(p, std::ios::binary);
  std::ostringstream b;
  b << in.rdbuf();
  return b.str();
}
std::filesystem::path temp_dir(const std::string& tag) {
  auto d = std::filesystem::temp_directory_path() / ("tlsph_b200_test_" + tag);
  std::filesystem::remove_all(d);
  std::filesystem::create_directories(d);
  return d;
}
}  // namespace

TEST_CASE("end_time = 0 produces only the initial probe sample") {  // test_runner.cpp:140-151
  ResolvedConfig cfg = parse_config(std::nullopt, {"case=bending_cantilever", "resolution=6", "end_time=0"});
  cfg.options.output_dir.clear();
  ProbeSeries series;
  const RunReport r = run_case(cfg, &series);
  CHECK(r.steps == 0);
  REQUIRE(series.samples.size() == 1);
  CHECK(series.samples[0].t == 0.0);
}

TEST_CASE("short damped run: deterministic seeds") {  // test_runner.cpp:176-200
  auto run_to_csv = [](std::uint64_t seed, const std::string& tag) {
    ResolvedConfig cfg = parse_config(
        std::nullopt, {"case=bending_cantilever", "resolution=6", "end_time=0.02", "damping.scheme=particle_split",
                       "damping.eta=32", "damping.alpha=0.2", "seed=" + std::to_string(seed), "output.snapshots=none"});
    const auto dir = temp_dir("det_" + tag);
    cfg.options.output_dir = dir.string();
    run_case(cfg);
    const std::string s = read_file((dir / "probe.csv").string());
    std::filesystem::remove_all(dir);
    return s;
  };
  const std::string a = run_to_csv(42, "a"), b = run_to_csv(42, "b"), c = run_to_csv(43, "c");
  CHECK(a == b);
  CHECK(a != c);
  CHECK(a.rfind("t,ux,uy,uz\n", 0) == 0);
}

TEST_CASE("damped step fraction tracks alpha and the report is consistent") {  // :202-225
  ResolvedConfig cfg =
      parse_config(std::nullopt, {"case=bending_cantilever", "resolution=6", "end_time=0.15",
                                  "damping.scheme=particle_split", "damping.eta=32", "damping.alpha=0.2", "seed=3"});
  cfg.options.output_dir.clear();
  const RunReport r = run_case(cfg);
  REQUIRE(r.steps > 100);
  const double n = static_cast<double>(r.steps);
  CHECK(std::abs(r.damped_steps / n - 0.2) <= 3.0 * std::sqrt(0.2 * 0.8 / n));
  CHECK(r.elastic_seconds + r.damping_seconds + r.neighbor_seconds <= r.total_seconds + 1e-9);
}

TEST_CASE("snapshots: initial stress-free, per-interval files, report json") {  // :153-174, :227-239
  ResolvedConfig cfg = parse_config(std::nullopt, {"case=bending_cantilever", "resolution=6", "end_time=0.012",
                                                   "output.interval=0.005", "output.snapshots=all"});
  const auto dir = temp_dir("snap");
  cfg.options.output_dir = dir.string();
  run_case(cfg);
  std::ifstream in(dir / "snapshot_initial.csv");
  REQUIRE(in.good());
  std::string line;
  std::getline(in, line);
  CHECK(line == "id,x,y,z,vx,vy,vz,von_mises");
  std::size_t rows = 0;
  while (std::getline(in, line)) {
    ++rows;
    CHECK(std::stod(line.substr(line.rfind(',') + 1)) == 0.0);
  }
  CHECK(rows == 18 * 6 * 6);
  CHECK(std::filesystem::exists(dir / "snapshot_000001.csv"));
  CHECK(std::filesystem::exists(dir / "snapshot_000002.csv"));
  CHECK(std::filesystem::exists(dir / "snapshot_final.csv"));
  const std::string rep = read_file((dir / "report.json").string());
  CHECK(rep.find("\"case\": \"bending_cantilever\"") != std::string::npos);
  std::filesystem::remove_all(dir);
}

TH_MAIN
