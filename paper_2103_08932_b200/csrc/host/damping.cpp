// Random-choice splitting damping through the device (reference:
// proj/src/tlsph/damping.cpp:12-182). Scalar helpers stay on the host; the
// operators run the sm_100a kernels on the device system kept resident for
// the caller's neighbourhood (resident.hpp), moving only v (and the masses and
// clamp flags the update reads) per call. Default ORDERED reductions:
// bit-identical to the reference arithmetic (tlsph/device.hpp).
#include "tlsph/damping.hpp"

#include <cmath>
#include <string>

#include "resident.hpp"
#include "tlsph/errors.hpp"

namespace tlsph {

double artificial_viscosity(double beta, double rho0, double E, double L) {
  require(beta >= 0.0 && rho0 > 0.0 && E > 0.0 && L > 0.0, ErrorKind::InvalidArgument,
          "artificial viscosity inputs must be positive");
  return 0.25 * beta * std::sqrt(rho0 * E) * L;
}

ViscousBounds viscous_dt_bounds(double h, double nu_kin, int dim) {
  require(h > 0.0 && nu_kin > 0.0, ErrorKind::InvalidArgument, "viscous bounds need positive h and viscosity");
  require(dim >= 1 && dim <= 3, ErrorKind::InvalidArgument, "dimension must be 1, 2 or 3");
  ViscousBounds b;
  b.explicit_bound = 0.5 * h * h / (nu_kin * dim);
  b.implicit_bound = 50.0 * h * h / (nu_kin * dim);
  return b;
}

double random_choice_eta(double eta, double alpha, RandomSource& rng) {
  require(alpha > 0.0 && alpha <= 1.0, ErrorKind::InvalidArgument,
          "random-choice probability must lie in (0, 1], got " + std::to_string(alpha));
  const double phi = rng.uniform();
  return phi < alpha ? eta / alpha : 0.0;
}

// Inputs of the local damping operators: v and the masses / clamp flags (damping.cpp:53-106).
template <int D>
void put_damping_inputs(tlsph_dev* dev, const ParticleSystem<D>& system) {
  host::put(dev, TLSPH_FIELD_V, system.v);
  host::refresh(dev, TLSPH_FIELD_M, system.m);
  host::refresh(dev, TLSPH_FIELD_CONSTRAINED, system.constrained);
}

template <int D>
void explicit_damping_accel(const ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh, double eta,
                            std::vector<Vec<D>>& out, int threads) {
  (void)threads;
  out.resize(system.size());
  auto lease = host::resident<D>(system, nbh, nullptr);
  put_damping_inputs<D>(lease.get(), system);
  static_assert(sizeof(Vec<D>) == D * sizeof(double));
  host::check(tlsph_dev_explicit_damping_accel(lease.get(), eta, reinterpret_cast<double*>(out.data())));
}

template <int D>
void particle_split_update(std::size_t i, ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh, double eta,
                           double dt_half) {
  auto lease = host::resident<D>(system, nbh, nullptr);
  put_damping_inputs<D>(lease.get(), system);
  host::check(tlsph_dev_particle_split_update(lease.get(), i, eta, dt_half));
  host::take(lease.get(), TLSPH_FIELD_V, system.v);
}

template <int D>
void pairwise_split_update(std::size_t i, std::int64_t slot, ParticleSystem<D>& system,
                           const ReferenceNeighborhood<D>& nbh, double eta, double dt_half) {
  auto lease = host::resident<D>(system, nbh, nullptr);
  put_damping_inputs<D>(lease.get(), system);
  host::check(tlsph_dev_pairwise_split_update(lease.get(), i, slot, eta, dt_half));
  host::take(lease.get(), TLSPH_FIELD_V, system.v);
}

// The sweep runs over the caller's grid: the resident system's cell order is checked against it
// once (build_cell_grid of the same r0 and cell size gives the same cells bit for bit).
template <int D>
void strang_damping_sweep(ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh, const CellGrid<D>& grid,
                          const BlockDecomposition<D>& blocks, DampingScheme scheme, double eta_tilde, double dt,
                          int threads) {
  (void)blocks;  // the colouring is implicit in the grid on the device
  (void)threads;
  if (eta_tilde == 0.0) return;
  require(scheme != DampingScheme::Explicit, ErrorKind::InvalidArgument,
          "the explicit scheme is integrated directly, not swept");
  auto lease = host::resident<D>(system, nbh, &grid);
  put_damping_inputs<D>(lease.get(), system);
  const auto s = scheme == DampingScheme::ParticleSplit ? TLSPH_SCHEME_PARTICLE_SPLIT : TLSPH_SCHEME_PAIRWISE_SPLIT;
  host::check(tlsph_dev_damping_sweep(lease.get(), s, eta_tilde, dt));
  host::take(lease.get(), TLSPH_FIELD_V, system.v);
}

#define TLSPH_INSTANTIATE(D)                                                                                    \
  template void explicit_damping_accel<D>(const ParticleSystem<D>&, const ReferenceNeighborhood<D>&, double,   \
                                          std::vector<Vec<D>>&, int);                                          \
  template void particle_split_update<D>(std::size_t, ParticleSystem<D>&, const ReferenceNeighborhood<D>&,      \
                                         double, double);                                                       \
  template void pairwise_split_update<D>(std::size_t, std::int64_t, ParticleSystem<D>&,                         \
                                         const ReferenceNeighborhood<D>&, double, double);                      \
  template void strang_damping_sweep<D>(ParticleSystem<D>&, const ReferenceNeighborhood<D>&, const CellGrid<D>&, \
                                        const BlockDecomposition<D>&, DampingScheme, double, double, int);
TLSPH_INSTANTIATE(2)
TLSPH_INSTANTIATE(3)
#undef TLSPH_INSTANTIATE

}  // namespace tlsph
