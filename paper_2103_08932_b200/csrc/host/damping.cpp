// Random-choice splitting damping through the device (reference:
// proj/src/tlsph/damping.cpp:12-182). Scalar helpers stay on the host; the
// operators upload the system and neighbourhood, run the sm_100a kernels in
// ORDERED mode (bit-identical to the reference arithmetic) and download v.
#include "tlsph/damping.hpp"

#include <cmath>
#include <string>

#include "devbridge.hpp"
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

template <int D>
void explicit_damping_accel(const ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh, double eta,
                            std::vector<Vec<D>>& out, int threads) {
  (void)threads;
  out.resize(system.size());
  auto h = host::upload<D>(system, nbh, host::coarse_cutoff<D>(system, nbh));
  host::put<D>(h.get(), TLSPH_FIELD_V, system.v);
  std::vector<double> flat(system.size() * D);
  host::check(tlsph_dev_explicit_damping_accel(h.get(), eta, flat.data()));
  host::unflatten<D>(flat, out);
}

template <int D>
void particle_split_update(std::size_t i, ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh, double eta,
                           double dt_half) {
  auto h = host::upload<D>(system, nbh, host::coarse_cutoff<D>(system, nbh));
  host::put<D>(h.get(), TLSPH_FIELD_V, system.v);
  host::check(tlsph_dev_particle_split_update(h.get(), i, eta, dt_half));
  host::get<D>(h.get(), TLSPH_FIELD_V, system.v);
}

template <int D>
void pairwise_split_update(std::size_t i, std::int64_t slot, ParticleSystem<D>& system,
                           const ReferenceNeighborhood<D>& nbh, double eta, double dt_half) {
  auto h = host::upload<D>(system, nbh, host::coarse_cutoff<D>(system, nbh));
  host::put<D>(h.get(), TLSPH_FIELD_V, system.v);
  host::check(tlsph_dev_pairwise_split_update(h.get(), i, slot, eta, dt_half));
  host::get<D>(h.get(), TLSPH_FIELD_V, system.v);
}

template <int D>
void strang_damping_sweep(ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh, const CellGrid<D>& grid,
                          const BlockDecomposition<D>& blocks, DampingScheme scheme, double eta_tilde, double dt,
                          int threads) {
  (void)blocks;  // the colouring is implicit in the grid on the device
  (void)threads;
  if (eta_tilde == 0.0) return;
  require(scheme != DampingScheme::Explicit, ErrorKind::InvalidArgument,
          "the explicit scheme is integrated directly, not swept");
  auto h = host::upload<D>(system, nbh, grid.cell_size);
  host::put<D>(h.get(), TLSPH_FIELD_V, system.v);
  const auto s = scheme == DampingScheme::ParticleSplit ? TLSPH_SCHEME_PARTICLE_SPLIT : TLSPH_SCHEME_PAIRWISE_SPLIT;
  host::check(tlsph_dev_damping_sweep(h.get(), s, eta_tilde, dt));
  host::get<D>(h.get(), TLSPH_FIELD_V, system.v);
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
