// TEST INFRASTRUCTURE ONLY — CPU oracle for the TL-SPH dynamic-relaxation hot path.
//
// This header is a plain C++20 (+ OpenMP) restatement of the reference's
// algorithm, written to be the parity checker and the CPU baseline. Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
// may load it. The product (paper_2103_08932_b200/) never links or calls it.
//
// Parity status: the reference itself cannot be compiled in this image (it
// needs Eigen3 and oneTBB, both absent). This oracle is
// pinned instead against every known-answer test the reference's own test
// suite holds for the path (tests/test_oracle_pins.py ports them), which is
// what SURVEY.md §8(c) lists.
//
// Each function cites the reference file:line it restates. Expressions keep
// the reference's evaluation order. Where the reference delegates arithmetic
// to Eigen (norm, determinant, inverse, small products) the order below is
// the Eigen 3.3/3.4 fixed-size code path (unpinned: Eigen is absent here):
//   * norm()          = sqrt((x0*x0 + x1*x1) + x2*x2)
//   * determinant 3x3 = m00*(m11*m22-m12*m21) - m01*(m10*m22-m12*m20) + m02*(m10*m21-m11*m20)
//   * inverse 3x3     = adjugate * (1/det) with det from the first cofactor column
//   * lazy products   = inner index ascending, ((p0+p1)+p2)
//   * s*(A*B)         = (s*A)*B  (Eigen's scalar-times-product rewrite)
// Compile with -ffp-contract=off (the reference Release build has no -march,
// so x86-64 baseline code never contracts to FMA).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace orc {

// ---------------------------------------------------------------- errors
// reference: proj/src/tlsph/errors.hpp:9-35
enum class ErrorKind { InvalidArgument = 1, Parse = 2, DegenerateGeometry = 3,
                       InvertedElement = 4, NumericalFailure = 5, Io = 6 };

struct Error : std::runtime_error {
  ErrorKind kind;
  Error(ErrorKind k, const std::string& m) : std::runtime_error(m), kind(k) {}
};

inline void require(bool ok, ErrorKind k, const std::string& msg) {
  if (!ok) throw Error(k, msg);
}

// ---------------------------------------------------------------- small fp64 types
// reference: proj/src/tlsph/math_types.hpp:8-21 (Eigen fixed-size aliases)
template <int D>
struct Vec {
  double c[D];
  static Vec zero() { Vec v; for (int d = 0; d < D; ++d) v.c[d] = 0.0; return v; }
  double& operator[](int d) { return c[d]; }
  double operator[](int d) const { return c[d]; }
};

template <int D>
struct Mat {
  double c[D][D];  // (row, col)
  static Mat zero() { Mat m; for (int r = 0; r < D; ++r) for (int k = 0; k < D; ++k) m.c[r][k] = 0.0; return m; }
  static Mat identity() { Mat m = zero(); for (int r = 0; r < D; ++r) m.c[r][r] = 1.0; return m; }
  double& operator()(int r, int k) { return c[r][k]; }
  double operator()(int r, int k) const { return c[r][k]; }
};

template <int D>
inline double squared_norm(const Vec<D>& v) {
  double s = v[0] * v[0];
  for (int d = 1; d < D; ++d) s = s + v[d] * v[d];
  return s;
}

template <int D>
inline double norm(const Vec<D>& v) { return std::sqrt(squared_norm(v)); }

// A*B with the inner index ascending.
template <int D>
inline Mat<D> matmul(const Mat<D>& a, const Mat<D>& b) {
  Mat<D> out;
  for (int r = 0; r < D; ++r)
    for (int k = 0; k < D; ++k) {
      double s = a(r, 0) * b(0, k);
      for (int q = 1; q < D; ++q) s = s + a(r, q) * b(q, k);
      out(r, k) = s;
    }
  return out;
}

template <int D>
inline Mat<D> transpose(const Mat<D>& a) {
  Mat<D> t;
  for (int r = 0; r < D; ++r) for (int k = 0; k < D; ++k) t(r, k) = a(k, r);
  return t;
}

inline double determinant(const Mat<2>& m) {
  return m(0, 0) * m(1, 1) - m(1, 0) * m(0, 1);
}

inline double determinant(const Mat<3>& m) {
  return m(0, 0) * (m(1, 1) * m(2, 2) - m(1, 2) * m(2, 1)) -
         m(0, 1) * (m(1, 0) * m(2, 2) - m(1, 2) * m(2, 0)) +
         m(0, 2) * (m(1, 0) * m(2, 1) - m(1, 1) * m(2, 0));
}

inline Mat<2> inverse(const Mat<2>& m) {
  const double invdet = 1.0 / determinant(m);
  Mat<2> r;
  r(0, 0) = m(1, 1) * invdet;
  r(1, 0) = -m(1, 0) * invdet;
  r(0, 1) = -m(0, 1) * invdet;
  r(1, 1) = m(0, 0) * invdet;
  return r;
}

// cofactor (i, j) with cyclic index arithmetic
inline double cofactor3(const Mat<3>& m, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return m(i1, j1) * m(i2, j2) - m(i1, j2) * m(i2, j1);
}

inline Mat<3> inverse(const Mat<3>& m) {
  const double c00 = cofactor3(m, 0, 0), c10 = cofactor3(m, 1, 0), c20 = cofactor3(m, 2, 0);
  const double det = (c00 * m(0, 0) + c10 * m(1, 0)) + c20 * m(2, 0);
  const double invdet = 1.0 / det;
  Mat<3> r;
  for (int row = 0; row < 3; ++row)
    for (int col = 0; col < 3; ++col) r(row, col) = cofactor3(m, col, row) * invdet;
  return r;
}

// Singular values (descending) of a small matrix by one-sided Jacobi
// rotations. Stands in for Eigen::JacobiSVD in the B0 condition check
// (integrator.cpp:27-31); only the boolean "smin > 0 && smax/smin <= 1e8"
// is consumed, so any accurate SVD is equivalent there. The device code uses
// the same routine so the boolean agrees bit for bit.
template <int D>
inline void singular_values(const Mat<D>& a, double* sv) {
  double u[D][D];
  for (int r = 0; r < D; ++r) for (int k = 0; k < D; ++k) u[r][k] = a(r, k);
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < D - 1; ++p)
      for (int q = p + 1; q < D; ++q) {
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        for (int r = 0; r < D; ++r) {
          alpha = alpha + u[r][p] * u[r][p];
          beta = beta + u[r][q] * u[r][q];
          gamma = gamma + u[r][p] * u[r][q];
        }
        if (gamma == 0.0 || std::fabs(gamma) <= 1e-300 ||
            std::fabs(gamma) <= 1e-17 * std::sqrt(alpha * beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t);
        const double sn = cs * t;
        for (int r = 0; r < D; ++r) {
          const double up = u[r][p], uq = u[r][q];
          u[r][p] = cs * up - sn * uq;
          u[r][q] = sn * up + cs * uq;
        }
      }
    if (!rotated) break;
  }
  for (int k = 0; k < D; ++k) {
    double s = 0.0;
    for (int r = 0; r < D; ++r) s = s + u[r][k] * u[r][k];
    sv[k] = std::sqrt(s);
  }
  std::sort(sv, sv + D, [](double x, double y) { return x > y; });
}

// ---------------------------------------------------------------- kernel
// reference: proj/src/tlsph/kernel.cpp:14-38 (Wendland C2)
constexpr double kPi = 3.14159265358979323846;

struct SmoothingKernel {
  double h, sigma;
  int dim;
  SmoothingKernel(double h_, int dim_) : h(h_), dim(dim_) {
    require(h_ > 0.0, ErrorKind::InvalidArgument, "smoothing length must be positive, got " + std::to_string(h_));
    require(dim_ == 2 || dim_ == 3, ErrorKind::InvalidArgument, "kernel dimension must be 2 or 3, got " + std::to_string(dim_));
    sigma = (dim_ == 2) ? 7.0 / (4.0 * kPi * h_ * h_) : 21.0 / (16.0 * kPi * h_ * h_ * h_);
  }
  double support_radius() const { return 2.0 * h; }
  double value(double r) const {
    require(r >= 0.0, ErrorKind::InvalidArgument, "kernel radius must be non-negative");
    const double q = r / h;
    if (q >= 2.0) return 0.0;
    const double t = 1.0 - 0.5 * q;
    const double t2 = t * t;
    return sigma * t2 * t2 * (1.0 + 2.0 * q);
  }
  double grad_mag(double r) const {
    require(r >= 0.0, ErrorKind::InvalidArgument, "kernel radius must be non-negative");
    const double q = r / h;
    if (q >= 2.0) return 0.0;
    const double t = 1.0 - 0.5 * q;
    return -5.0 * q * (sigma / h) * t * t * t;
  }
};

// ---------------------------------------------------------------- material
// reference: proj/src/tlsph/material.cpp:10-44, material.hpp:16-39
enum class Model { LinearKirchhoff = 0, NeoHookean = 1 };

struct Material {
  Model model = Model::LinearKirchhoff;
  double lambda = 0, mu = 0, K = 0, G = 0, E = 0, nu = 0, rho0 = 0, c = 0;
};

inline Material material_from_young_poisson(double E, double nu, double rho0, Model model) {
  require(E > 0.0, ErrorKind::InvalidArgument, "Young's modulus must be positive, got " + std::to_string(E));
  require(nu >= 0.0 && nu < 0.5, ErrorKind::InvalidArgument, "Poisson ratio must lie in [0, 0.5), got " + std::to_string(nu));
  require(rho0 > 0.0, ErrorKind::InvalidArgument, "reference density must be positive, got " + std::to_string(rho0));
  Material m;
  m.model = model; m.E = E; m.nu = nu; m.rho0 = rho0;
  m.mu = E / (2.0 * (1.0 + nu));
  m.lambda = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  m.K = m.lambda + 2.0 * m.mu / 3.0;
  m.G = m.mu;
  m.c = std::sqrt(m.K / rho0);
  return m;
}

template <int D>
inline Mat<D> second_pk(const Mat<D>& F, const Material& mat) {
  const double J = determinant(F);
  require(J > 0.0, ErrorKind::InvertedElement,
          "deformation gradient has non-positive determinant " + std::to_string(J));
  const Mat<D> C = matmul(transpose(F), F);
  Mat<D> S;
  if (mat.model == Model::LinearKirchhoff) {
    Mat<D> g;
    for (int r = 0; r < D; ++r) for (int k = 0; k < D; ++k) g(r, k) = 0.5 * (C(r, k) - (r == k ? 1.0 : 0.0));
    double tr = g(0, 0);
    for (int d = 1; d < D; ++d) tr = tr + g(d, d);
    const double lt = mat.lambda * tr;
    const double twomu = 2.0 * mat.mu;
    for (int r = 0; r < D; ++r) for (int k = 0; k < D; ++k) S(r, k) = lt * (r == k ? 1.0 : 0.0) + twomu * g(r, k);
    return S;
  }
  const Mat<D> Ci = inverse(C);
  const double ll = mat.lambda * std::log(J);
  for (int r = 0; r < D; ++r)
    for (int k = 0; k < D; ++k) S(r, k) = mat.mu * ((r == k ? 1.0 : 0.0) - Ci(r, k)) + ll * Ci(r, k);
  return S;
}

// ---------------------------------------------------------------- state
// reference: proj/src/tlsph/particle_system.hpp:15-59
template <int D>
struct ParticleSystem {
  std::vector<Vec<D>> r0, r, v, a;
  std::vector<Mat<D>> F, dFdt, B0;
  std::vector<double> V0, m, rho0, rho;
  std::vector<std::uint8_t> constrained;
  std::size_t size() const { return r0.size(); }
  void add_particle(const Vec<D>& p, double volume, double density) {
    r0.push_back(p); r.push_back(p);
    v.push_back(Vec<D>::zero()); a.push_back(Vec<D>::zero());
    F.push_back(Mat<D>::identity()); dFdt.push_back(Mat<D>::zero()); B0.push_back(Mat<D>::identity());
    V0.push_back(volume); m.push_back(density * volume); rho0.push_back(density); rho.push_back(density);
    constrained.push_back(0);
  }
  void apply_constraints() {
    for (std::size_t i = 0; i < size(); ++i)
      if (constrained[i]) { v[i] = Vec<D>::zero(); r[i] = r0[i]; }
  }
};

// ---------------------------------------------------------------- parallel helper
// reference: proj/src/tlsph/parallel.hpp:14-27 (TBB arena per call -> OpenMP team)
template <typename Body>
inline void parallel_for_range(std::size_t n, int threads, Body&& body) {
  if (threads <= 1 || n < 2) { body(std::size_t{0}, n); return; }
#ifdef _OPENMP
  const long long nn = static_cast<long long>(n);
  const long long chunk = 256;
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1)
  for (long long lo = 0; lo < nn; lo += chunk) {
    const long long hi = std::min(nn, lo + chunk);
    body(static_cast<std::size_t>(lo), static_cast<std::size_t>(hi));
  }
#else
  body(std::size_t{0}, n);
#endif
}

// ---------------------------------------------------------------- neighbours
// reference: proj/src/tlsph/neighbors.hpp:18-48, neighbors.cpp:14-59
template <int D>
struct CellGrid {
  Vec<D> origin = Vec<D>::zero();
  double cell_size = 0.0;
  std::array<int, D> dims{};
  std::vector<int> cell_of;
  std::vector<std::vector<int>> cells;
  int cell_count() const { int n = 1; for (int d = 0; d < D; ++d) n *= dims[d]; return n; }
  int linear_index(const std::array<int, D>& c) const {
    int idx = c[D - 1];
    for (int d = D - 2; d >= 0; --d) idx = idx * dims[d] + c[d];
    return idx;
  }
  std::array<int, D> coords_of(int linear) const {
    std::array<int, D> c{};
    for (int d = 0; d < D; ++d) { c[d] = linear % dims[d]; linear /= dims[d]; }
    return c;
  }
  std::array<int, D> coords_of_position(const Vec<D>& p) const {
    std::array<int, D> c{};
    for (int d = 0; d < D; ++d) {
      const int idx = static_cast<int>(std::floor((p[d] - origin[d]) / cell_size));
      c[d] = std::clamp(idx, 0, dims[d] - 1);
    }
    return c;
  }
};

template <int D>
inline CellGrid<D> build_cell_grid(const std::vector<Vec<D>>& pos, double cutoff) {
  require(!pos.empty(), ErrorKind::InvalidArgument, "cell grid needs at least one particle");
  require(cutoff > 0.0, ErrorKind::InvalidArgument, "cell grid cutoff must be positive");
  Vec<D> lo = pos[0], hi = pos[0];
  for (const auto& p : pos)
    for (int d = 0; d < D; ++d) {
      require(std::isfinite(p[d]), ErrorKind::InvalidArgument, "non-finite particle position");
      lo[d] = std::min(lo[d], p[d]);
      hi[d] = std::max(hi[d], p[d]);
    }
  CellGrid<D> g;
  g.cell_size = cutoff;
  g.origin = lo;
  for (int d = 0; d < D; ++d) {
    const double extent = hi[d] - lo[d];
    g.dims[d] = std::max(1, static_cast<int>(std::floor(extent / cutoff)) + 1);
  }
  g.cells.assign(static_cast<std::size_t>(g.cell_count()), {});
  g.cell_of.resize(pos.size());
  for (std::size_t i = 0; i < pos.size(); ++i) {
    const int cell = g.linear_index(g.coords_of_position(pos[i]));
    g.cell_of[i] = cell;
    g.cells[static_cast<std::size_t>(cell)].push_back(static_cast<int>(i));
  }
  return g;
}

// reference: neighbors.cpp:61-77 (3-per-axis residue colouring)
template <int D>
inline std::vector<std::vector<int>> block_decompose(const CellGrid<D>& g) {
  std::vector<std::vector<int>> blocks(D == 2 ? 9 : 27);
  for (int cell = 0; cell < g.cell_count(); ++cell) {
    const auto c = g.coords_of(cell);
    int b = 0, stride = 1;
    for (int d = 0; d < D; ++d) { b += (c[d] % 3) * stride; stride *= 3; }
    blocks[static_cast<std::size_t>(b)].push_back(cell);
  }
  return blocks;
}

// reference: neighbors.hpp:67-82
template <int D>
struct Neighborhood {
  std::vector<std::int64_t> offsets;
  std::vector<int> neighbor;
  std::vector<double> r0_len;
  std::vector<Vec<D>> e0;
  std::vector<double> dwdr0;
  std::vector<double> pair_factor;
  std::int64_t begin(std::size_t i) const { return offsets[i]; }
  std::int64_t end(std::size_t i) const { return offsets[i + 1]; }
  std::size_t count(std::size_t i) const { return static_cast<std::size_t>(offsets[i + 1] - offsets[i]); }
};

// reference: neighbors.cpp:79-141. The per-particle scans are independent, so the checker runs
// them on an OpenMP team (`threads`, default all): the lists, slot values and the error (the
// coincident pair the serial loop meets first: lowest i, then that i's first j in stencil order)
// are those of the reference's serial loop.
template <int D>
inline Neighborhood<D> build_reference_neighborhoods(const std::vector<Vec<D>>& r0,
                                                     const std::vector<double>& V0,
                                                     const SmoothingKernel& kernel,
                                                     const CellGrid<D>& grid, int threads = 0) {
  const std::size_t n = r0.size();
  require(V0.size() == n, ErrorKind::InvalidArgument, "volume array size does not match particle count");
  if (threads <= 0) threads = omp_get_max_threads();
  const double cutoff = kernel.support_radius();
  Neighborhood<D> nbh;
  nbh.offsets.assign(n + 1, 0);
  std::vector<std::vector<int>> lists(n);
  std::vector<int> coincident(n, -1);  // first coincident j of particle i (-1: none)
  parallel_for_range(n, threads, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      const auto base = grid.coords_of_position(r0[i]);
      std::array<int, D> c{};
      const int stencil = (D == 2) ? 9 : 27;
      for (int s = 0; s < stencil && coincident[i] < 0; ++s) {
        int rem = s;
        bool in_range = true;
        for (int d = 0; d < D; ++d) {
          c[d] = base[d] + (rem % 3) - 1;
          rem /= 3;
          if (c[d] < 0 || c[d] >= grid.dims[d]) in_range = false;
        }
        if (!in_range) continue;
        for (int j : grid.cells[static_cast<std::size_t>(grid.linear_index(c))]) {
          if (static_cast<std::size_t>(j) == i) continue;
          Vec<D> diff;
          for (int d = 0; d < D; ++d) diff[d] = r0[i][d] - r0[static_cast<std::size_t>(j)][d];
          const double dist = norm(diff);
          if (dist >= cutoff) continue;
          if (!(dist > 0.0)) {
            coincident[i] = j;
            break;
          }
          lists[i].push_back(j);
        }
      }
      std::sort(lists[i].begin(), lists[i].end());
    }
  });
  for (std::size_t i = 0; i < n; ++i) {
    require(coincident[i] < 0, ErrorKind::DegenerateGeometry,
            "coincident particles " + std::to_string(i) + " and " + std::to_string(coincident[i]) +
                " in reference configuration");
    nbh.offsets[i + 1] = nbh.offsets[i] + static_cast<std::int64_t>(lists[i].size());
  }
  const std::size_t total = static_cast<std::size_t>(nbh.offsets[n]);
  nbh.neighbor.resize(total); nbh.r0_len.resize(total); nbh.e0.resize(total);
  nbh.dwdr0.resize(total); nbh.pair_factor.resize(total);
  parallel_for_range(n, threads, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      std::int64_t slot = nbh.offsets[i];
      for (int j : lists[i]) {
        Vec<D> diff;
        for (int d = 0; d < D; ++d) diff[d] = r0[i][d] - r0[static_cast<std::size_t>(j)][d];
        const double dist = norm(diff);
        const double dw = kernel.grad_mag(dist);
        nbh.neighbor[static_cast<std::size_t>(slot)] = j;
        nbh.r0_len[static_cast<std::size_t>(slot)] = dist;
        Vec<D> e;
        for (int d = 0; d < D; ++d) e[d] = diff[d] / dist;
        nbh.e0[static_cast<std::size_t>(slot)] = e;
        nbh.dwdr0[static_cast<std::size_t>(slot)] = dw;
        nbh.pair_factor[static_cast<std::size_t>(slot)] = 2.0 * V0[i] * V0[static_cast<std::size_t>(j)] * dw / dist;
        ++slot;
      }
      std::vector<int>().swap(lists[i]);
    }
  });
  return nbh;
}

enum class SweepDirection { Forward, Reverse };

// reference: neighbors.cpp:143-174 (colours in sequence, same-colour cells concurrent)
template <typename CellTask>
inline void block_sweep(const std::vector<std::vector<int>>& blocks, const CellTask& task,
                        bool forward_then_reverse, int threads) {
  auto run_pass = [&](SweepDirection dir) {
    const int nb = static_cast<int>(blocks.size());
    for (int b = 0; b < nb; ++b) {
      const auto& cells = blocks[static_cast<std::size_t>(dir == SweepDirection::Forward ? b : nb - 1 - b)];
      if (cells.empty()) continue;
      const long long nc = static_cast<long long>(cells.size());
      auto run_cell = [&](long long k) {
        const long long idx = dir == SweepDirection::Forward ? k : nc - 1 - k;
        task(cells[static_cast<std::size_t>(idx)], dir);
      };
      if (threads <= 1 || nc < 2) {
        for (long long k = 0; k < nc; ++k) run_cell(k);
      } else {
#ifdef _OPENMP
#pragma omp parallel for num_threads(threads) schedule(dynamic, 4)
        for (long long k = 0; k < nc; ++k) run_cell(k);
#else
        for (long long k = 0; k < nc; ++k) run_cell(k);
#endif
      }
    }
  };
  run_pass(SweepDirection::Forward);
  if (forward_then_reverse) run_pass(SweepDirection::Reverse);
}

// ---------------------------------------------------------------- damping
// reference: proj/src/tlsph/damping.hpp:12-91, damping.cpp:12-182
enum class Scheme { Explicit = 0, ParticleSplit = 1, PairwiseSplit = 2 };

inline double artificial_viscosity(double beta, double rho0, double E, double L) {
  require(beta >= 0.0 && rho0 > 0.0 && E > 0.0 && L > 0.0, ErrorKind::InvalidArgument,
          "artificial viscosity inputs must be positive");
  return 0.25 * beta * std::sqrt(rho0 * E) * L;
}

struct ViscousBounds { double explicit_bound = 0.0, implicit_bound = 0.0; };

inline ViscousBounds viscous_dt_bounds(double h, double nu_kin, int dim) {
  require(h > 0.0 && nu_kin > 0.0, ErrorKind::InvalidArgument, "viscous bounds need positive h and viscosity");
  require(dim >= 1 && dim <= 3, ErrorKind::InvalidArgument, "dimension must be 1, 2 or 3");
  ViscousBounds b;
  b.explicit_bound = 0.5 * h * h / (nu_kin * dim);
  b.implicit_bound = 50.0 * h * h / (nu_kin * dim);
  return b;
}

// reference: damping.hpp:41-50 — std::mt19937_64, u = (x >> 11) * 2^-53
struct RandomSource {
  std::mt19937_64 gen;
  explicit RandomSource(std::uint64_t seed) : gen(seed) {}
  double uniform() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
};

// reference: damping.cpp:29-34
inline double random_choice_eta(double eta, double alpha, RandomSource& rng) {
  require(alpha > 0.0 && alpha <= 1.0, ErrorKind::InvalidArgument,
          "random-choice probability must lie in (0, 1], got " + std::to_string(alpha));
  const double phi = rng.uniform();
  return phi < alpha ? eta / alpha : 0.0;
}

// reference: damping.cpp:36-51
template <int D>
inline void explicit_damping_accel(const ParticleSystem<D>& sys, const Neighborhood<D>& nbh, double eta,
                                   std::vector<Vec<D>>& out, int threads) {
  out.resize(sys.size());
  parallel_for_range(sys.size(), threads, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      Vec<D> acc = Vec<D>::zero();
      for (auto s = nbh.begin(i); s < nbh.end(i); ++s) {
        const auto j = static_cast<std::size_t>(nbh.neighbor[static_cast<std::size_t>(s)]);
        const double g = nbh.pair_factor[static_cast<std::size_t>(s)];
        for (int d = 0; d < D; ++d) acc[d] = acc[d] + g * (sys.v[i][d] - sys.v[j][d]);
      }
      const double k = eta / sys.m[i];
      for (int d = 0; d < D; ++d) out[i][d] = k * acc[d];
    }
  });
}

// reference: damping.cpp:53-89
template <int D>
inline void particle_split_update(std::size_t i, ParticleSystem<D>& sys, const Neighborhood<D>& nbh,
                                  double eta, double dt_half) {
  const auto lo = nbh.begin(i), hi = nbh.end(i);
  if (lo == hi) return;
  Vec<D> residual = Vec<D>::zero();
  double sum_b = 0.0, sum_b2 = 0.0;
  for (auto s = lo; s < hi; ++s) {
    const auto j = static_cast<std::size_t>(nbh.neighbor[static_cast<std::size_t>(s)]);
    const double b = eta * nbh.pair_factor[static_cast<std::size_t>(s)] * dt_half;
    for (int d = 0; d < D; ++d) residual[d] = residual[d] - b * (sys.v[i][d] - sys.v[j][d]);
    sum_b = sum_b + b;
    sum_b2 = sum_b2 + b * b;
  }
  const double diag = sum_b - sys.m[i];
  const double denom = diag * diag + sum_b2;
  Vec<D> rate, vnew;
  for (int d = 0; d < D; ++d) rate[d] = residual[d] / denom;
  for (int d = 0; d < D; ++d) vnew[d] = sys.v[i][d] + diag * rate[d];
  for (auto s = lo; s < hi; ++s) {
    const auto j = static_cast<std::size_t>(nbh.neighbor[static_cast<std::size_t>(s)]);
    const double b = eta * nbh.pair_factor[static_cast<std::size_t>(s)] * dt_half;
    Vec<D> pred;
    for (int d = 0; d < D; ++d) pred[d] = sys.v[j][d] - b * rate[d];
    if (!sys.constrained[j]) {
      const double bm = b / sys.m[j];
      for (int d = 0; d < D; ++d) sys.v[j][d] = sys.v[j][d] - bm * (vnew[d] - pred[d]);
    }
  }
  sys.v[i] = vnew;
}

// reference: damping.cpp:91-106
template <int D>
inline void pairwise_split_update(std::size_t i, std::int64_t slot, ParticleSystem<D>& sys,
                                  const Neighborhood<D>& nbh, double eta, double dt_half) {
  const auto j = static_cast<std::size_t>(nbh.neighbor[static_cast<std::size_t>(slot)]);
  const double b = eta * nbh.pair_factor[static_cast<std::size_t>(slot)] * dt_half;
  const double mi = sys.m[i], mj = sys.m[j];
  const double denom = mi * mj - (mi + mj) * b;
  const double k = b / denom;
  Vec<D> scaled;
  for (int d = 0; d < D; ++d) scaled[d] = k * (sys.v[i][d] - sys.v[j][d]);
  for (int d = 0; d < D; ++d) sys.v[i][d] = sys.v[i][d] + mj * scaled[d];
  if (!sys.constrained[j])
    for (int d = 0; d < D; ++d) sys.v[j][d] = sys.v[j][d] - mi * scaled[d];
}

// reference: damping.cpp:125-182
template <int D>
inline void strang_damping_sweep(ParticleSystem<D>& sys, const Neighborhood<D>& nbh, const CellGrid<D>& grid,
                                 const std::vector<std::vector<int>>& blocks, Scheme scheme,
                                 double eta_tilde, double dt, int threads) {
  if (eta_tilde == 0.0) return;
  require(scheme != Scheme::Explicit, ErrorKind::InvalidArgument,
          "the explicit scheme is integrated directly, not swept");
  const double dt_half = 0.5 * dt;
  if (scheme == Scheme::ParticleSplit) {
    auto task = [&](int cell, SweepDirection dir) {
      const auto& ps = grid.cells[static_cast<std::size_t>(cell)];
      const std::size_t np = ps.size();
      for (std::size_t k = 0; k < np; ++k) {
        const auto i = static_cast<std::size_t>(ps[dir == SweepDirection::Forward ? k : np - 1 - k]);
        if (sys.constrained[i]) continue;
        particle_split_update(i, sys, nbh, eta_tilde, dt_half);
      }
    };
    block_sweep(blocks, task, true, threads);
  } else {
    const double dt_pair = 0.5 * dt_half;
    auto task = [&](int cell, SweepDirection dir) {
      const auto& ps = grid.cells[static_cast<std::size_t>(cell)];
      const std::size_t np = ps.size();
      for (std::size_t k = 0; k < np; ++k) {
        const auto i = static_cast<std::size_t>(ps[dir == SweepDirection::Forward ? k : np - 1 - k]);
        if (sys.constrained[i]) continue;
        const auto lo = nbh.begin(i), hi = nbh.end(i);
        for (auto s = lo; s < hi; ++s) pairwise_split_update(i, s, sys, nbh, eta_tilde, dt_pair);
        for (auto s = hi; s-- > lo;) pairwise_split_update(i, s, sys, nbh, eta_tilde, dt_pair);
      }
    };
    block_sweep(blocks, task, true, threads);
  }
}

// ---------------------------------------------------------------- integrator
// reference: proj/src/tlsph/integrator.cpp:12-42
template <int D>
inline void compute_correction_matrices(ParticleSystem<D>& sys, const Neighborhood<D>& nbh, int threads) {
  const std::size_t n = sys.size();
  std::vector<int> degenerate(n, 0);
  parallel_for_range(n, threads, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      Mat<D> moment = Mat<D>::zero();
      for (auto s = nbh.begin(i); s < nbh.end(i); ++s) {
        const auto ss = static_cast<std::size_t>(s);
        const auto j = static_cast<std::size_t>(nbh.neighbor[ss]);
        const double w = -sys.V0[j] * nbh.dwdr0[ss] * nbh.r0_len[ss];
        const Vec<D>& e = nbh.e0[ss];
        for (int r = 0; r < D; ++r) {
          const double we = w * e[r];
          for (int k = 0; k < D; ++k) moment(r, k) = moment(r, k) + we * e[k];
        }
      }
      double sv[D];
      singular_values(moment, sv);
      if (!(sv[D - 1] > 0.0) || sv[0] / sv[D - 1] > 1e8) { degenerate[i] = 1; continue; }
      sys.B0[i] = inverse(moment);
    }
  });
  for (std::size_t i = 0; i < n; ++i)
    require(!degenerate[i], ErrorKind::DegenerateGeometry,
            "degenerate neighborhood: correction matrix of particle " + std::to_string(i) +
                " is singular or ill-conditioned");
}

// reference: integrator.cpp:44-58
template <int D>
inline void compute_deformation_rate(ParticleSystem<D>& sys, const Neighborhood<D>& nbh, int threads) {
  parallel_for_range(sys.size(), threads, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      Mat<D> rate = Mat<D>::zero();
      for (auto s = nbh.begin(i); s < nbh.end(i); ++s) {
        const auto ss = static_cast<std::size_t>(s);
        const auto j = static_cast<std::size_t>(nbh.neighbor[ss]);
        const double k = sys.V0[j] * nbh.dwdr0[ss];
        const Vec<D>& e = nbh.e0[ss];
        for (int r = 0; r < D; ++r) {
          const double kv = k * (sys.v[i][r] - sys.v[j][r]);
          for (int q = 0; q < D; ++q) rate(r, q) = rate(r, q) - kv * e[q];
        }
      }
      sys.dFdt[i] = matmul(rate, sys.B0[i]);
    }
  });
}

// reference: integrator.cpp:60-78
template <int D>
inline void update_density(ParticleSystem<D>& sys, int threads) {
  const std::size_t n = sys.size();
  std::vector<int> inverted(n, 0);
  parallel_for_range(n, threads, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      const double J = determinant(sys.F[i]);
      if (!(J > 0.0)) { inverted[i] = 1; continue; }
      sys.rho[i] = sys.rho0[i] / J;
    }
  });
  for (std::size_t i = 0; i < n; ++i)
    require(!inverted[i], ErrorKind::InvertedElement,
            "inverted element: det(F) <= 0 for particle " + std::to_string(i));
}

// reference: forces.hpp:13-39 -- the per-particle body term plus the optional penalty contact
// plane of the falling-ball case, evaluated at the current position:
// gap = (r - point).normal; gap < 0 adds (stiffness * (-gap) / m) * normal.
template <int D>
struct ExternalAccel {
  std::vector<Vec<D>> body;  // empty = zero
  bool contact = false;
  Vec<D> cp_point = Vec<D>::zero(), cp_normal = Vec<D>::zero();
  double cp_k = 0.0;
  Vec<D> eval(std::size_t i, const Vec<D>& r, double m) const {
    Vec<D> acc = body.empty() ? Vec<D>::zero() : body[i];
    if (!contact) return acc;
    double gap = (r[0] - cp_point[0]) * cp_normal[0];
    for (int d = 1; d < D; ++d) gap = gap + (r[d] - cp_point[d]) * cp_normal[d];
    if (gap >= 0.0) return acc;
    const double k = cp_k * (-gap) / m;
    for (int d = 0; d < D; ++d) acc[d] = acc[d] + k * cp_normal[d];
    return acc;
  }
};

// reference: integrator.cpp:80-116
template <int D>
inline void compute_momentum_rhs(ParticleSystem<D>& sys, const Neighborhood<D>& nbh, const Material& mat,
                                 const ExternalAccel<D>& ext, int threads) {
  const std::size_t n = sys.size();
  std::vector<Mat<D>> st(n);
  std::vector<int> inverted(n, 0);
  parallel_for_range(n, threads, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      if (!(determinant(sys.F[i]) > 0.0)) { inverted[i] = 1; st[i] = Mat<D>::zero(); continue; }
      const Mat<D> S = second_pk<D>(sys.F[i], mat);
      st[i] = matmul(matmul(sys.F[i], S), sys.B0[i]);
    }
  });
  for (std::size_t i = 0; i < n; ++i)
    require(!inverted[i], ErrorKind::InvertedElement,
            "inverted element: det(F) <= 0 for particle " + std::to_string(i));
  parallel_for_range(n, threads, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      Vec<D> acc = Vec<D>::zero();
      for (auto s = nbh.begin(i); s < nbh.end(i); ++s) {
        const auto ss = static_cast<std::size_t>(s);
        const auto j = static_cast<std::size_t>(nbh.neighbor[ss]);
        const double k = sys.V0[i] * sys.V0[j] * nbh.dwdr0[ss];
        const Vec<D>& e = nbh.e0[ss];
        for (int r = 0; r < D; ++r) {
          double t = (k * (st[i](r, 0) + st[j](r, 0))) * e[0];
          for (int q = 1; q < D; ++q) t = t + (k * (st[i](r, q) + st[j](r, q))) * e[q];
          acc[r] = acc[r] + t;
        }
      }
      const Vec<D> g = ext.eval(i, sys.r[i], sys.m[i]);
      for (int d = 0; d < D; ++d) sys.a[i][d] = acc[d] / sys.m[i] + g[d];
    }
  });
}

// reference: integrator.cpp:118-152
template <int D>
inline void verlet_step(ParticleSystem<D>& sys, const Neighborhood<D>& nbh, const Material& mat,
                        const ExternalAccel<D>& ext, double dt, int threads) {
  const std::size_t n = sys.size();
  const double half = 0.5 * dt;
  update_density(sys, threads);
  parallel_for_range(n, threads, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      for (int r = 0; r < D; ++r) for (int q = 0; q < D; ++q) sys.F[i](r, q) = sys.F[i](r, q) + half * sys.dFdt[i](r, q);
      for (int d = 0; d < D; ++d) sys.r[i][d] = sys.r[i][d] + half * sys.v[i][d];
    }
  });
  sys.apply_constraints();
  compute_momentum_rhs(sys, nbh, mat, ext, threads);
  parallel_for_range(n, threads, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i)
      for (int d = 0; d < D; ++d) sys.v[i][d] = sys.v[i][d] + dt * sys.a[i][d];
  });
  sys.apply_constraints();
  compute_deformation_rate(sys, nbh, threads);
  update_density(sys, threads);
  parallel_for_range(n, threads, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      for (int r = 0; r < D; ++r) for (int q = 0; q < D; ++q) sys.F[i](r, q) = sys.F[i](r, q) + half * sys.dFdt[i](r, q);
      for (int d = 0; d < D; ++d) sys.r[i][d] = sys.r[i][d] + half * sys.v[i][d];
    }
  });
  sys.apply_constraints();
}

// reference: integrator.cpp:154-169
template <int D>
inline double stable_dt(const ParticleSystem<D>& sys, const Material& mat, double h) {
  double vmax = 0.0, amax = 0.0;
  for (std::size_t i = 0; i < sys.size(); ++i) {
    vmax = std::max(vmax, norm(sys.v[i]));
    amax = std::max(amax, norm(sys.a[i]));
  }
  double bound = h / (mat.c + vmax);
  if (amax > 0.0) bound = std::min(bound, std::sqrt(h / amax));
  return 0.6 * bound;
}

// reference: integrator.cpp:171-178
template <int D>
inline double total_kinetic_energy(const ParticleSystem<D>& sys) {
  double e = 0.0;
  for (std::size_t i = 0; i < sys.size(); ++i) e = e + 0.5 * sys.m[i] * squared_norm(sys.v[i]);
  return e;
}

// reference: runner.cpp:233-247
template <int D>
inline void check_finite(const ParticleSystem<D>& sys, std::uint64_t step) {
  double total = 0.0;
  for (std::size_t i = 0; i < sys.size(); ++i) total = total + (squared_norm(sys.v[i]) + squared_norm(sys.r[i]));
  if (std::isfinite(total)) return;
  for (std::size_t i = 0; i < sys.size(); ++i) {
    bool fin = true;
    for (int d = 0; d < D; ++d) fin = fin && std::isfinite(sys.v[i][d]) && std::isfinite(sys.r[i][d]);
    if (!fin)
      throw Error(ErrorKind::NumericalFailure,
                  "NaN detected at step " + std::to_string(step) + ", particle " + std::to_string(i));
  }
}

// ---------------------------------------------------------------- scenarios
// reference: proj/src/tlsph/cases.cpp:21-46
template <int D>
inline void generate_box_lattice(ParticleSystem<D>& sys, const Vec<D>& lo, const Vec<D>& hi, double dp, double rho0) {
  require(dp > 0.0, ErrorKind::InvalidArgument, "lattice spacing must be positive");
  std::array<int, D> counts{};
  for (int d = 0; d < D; ++d) {
    const double extent = hi[d] - lo[d];
    require(extent >= dp * (1.0 - 1e-12), ErrorKind::InvalidArgument, "degenerate lattice dimension " + std::to_string(d));
    counts[d] = std::max(1, static_cast<int>(std::lround(extent / dp)));
  }
  const double volume = std::pow(dp, D);
  std::array<int, D> idx{};
  while (true) {
    Vec<D> p;
    for (int d = 0; d < D; ++d) p[d] = lo[d] + (idx[d] + 0.5) * dp;
    sys.add_particle(p, volume, rho0);
    int d = 0;
    for (; d < D; ++d) {
      if (++idx[d] < counts[d]) break;
      idx[d] = 0;
    }
    if (d == D) break;
  }
}

}  // namespace orc
