// TL-SPH operators through the device (reference: proj/src/tlsph/integrator.cpp:12-188).
#include "tlsph/integrator.hpp"

#include <cmath>
#include <string>

#include "devbridge.hpp"
#include "tlsph/errors.hpp"

namespace tlsph {

namespace {

template <int D>
void put_external(tlsph_dev* dev, const ParticleSystem<D>& system, const ExternalAccel<D>& ext) {
  if (!ext.body.empty()) {
    require(ext.body.size() == system.size(), ErrorKind::InvalidArgument, "body force size mismatch");
    host::put<D>(dev, TLSPH_FIELD_BODY, ext.body);
  }
  if (ext.contact) {
    double p[3] = {0, 0, 0}, nrm[3] = {0, 0, 0};
    for (int d = 0; d < D; ++d) {
      p[d] = ext.contact->point[d];
      nrm[d] = ext.contact->normal[d];
    }
    host::check(tlsph_dev_set_contact_plane(dev, p, nrm, ext.contact->stiffness));
  }
}

}  // namespace

template <int D>
void compute_correction_matrices(ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh, int threads) {
  (void)threads;
  auto h = host::upload<D>(system, nbh, host::coarse_cutoff<D>(system, nbh));
  host::put<D>(h.get(), TLSPH_FIELD_B0, system.B0);
  host::check(tlsph_dev_correction_matrices(h.get()));
  host::get<D>(h.get(), TLSPH_FIELD_B0, system.B0);
}

template <int D>
void compute_deformation_rate(ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh, int threads) {
  (void)threads;
  auto h = host::upload<D>(system, nbh, host::coarse_cutoff<D>(system, nbh));
  host::put<D>(h.get(), TLSPH_FIELD_V, system.v);
  host::put<D>(h.get(), TLSPH_FIELD_B0, system.B0);
  host::check(tlsph_dev_deformation_rate(h.get()));
  host::get<D>(h.get(), TLSPH_FIELD_DFDT, system.dFdt);
}

template <int D>
void update_density(ParticleSystem<D>& system, int threads) {
  (void)threads;
  ReferenceNeighborhood<D> empty;
  empty.offsets.assign(system.size() + 1, 0);
  auto h = host::upload<D>(system, empty, host::coarse_cutoff<D>(system, empty));
  host::put<D>(h.get(), TLSPH_FIELD_F, system.F);
  host::put(h.get(), TLSPH_FIELD_RHO, system.rho);
  const tlsph_status st = tlsph_dev_update_density(h.get());
  const std::string msg = tlsph_dev_last_error();
  host::get(h.get(), TLSPH_FIELD_RHO, system.rho);  // non-inverted particles are updated before the throw
  if (st == TLSPH_ERR_INVERTED_ELEMENT) throw Error(ErrorKind::InvertedElement, msg);
  host::check(st);
}

template <int D>
void compute_momentum_rhs(ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh, const Material& material,
                          const ExternalAccel<D>& external, int threads) {
  (void)threads;
  auto h = host::upload<D>(system, nbh, host::coarse_cutoff<D>(system, nbh));
  host::put<D>(h.get(), TLSPH_FIELD_F, system.F);
  host::put<D>(h.get(), TLSPH_FIELD_B0, system.B0);
  host::put<D>(h.get(), TLSPH_FIELD_R, system.r);
  put_external<D>(h.get(), system, external);
  const auto mat = host::to_dev(material);
  host::check(tlsph_dev_momentum_rhs(h.get(), &mat));
  host::get<D>(h.get(), TLSPH_FIELD_A, system.a);
}

template <int D>
void verlet_step(ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh, const Material& material,
                 const ExternalAccel<D>& external, double dt, int threads) {
  (void)threads;
  auto h = host::upload<D>(system, nbh, host::coarse_cutoff<D>(system, nbh));
  host::put<D>(h.get(), TLSPH_FIELD_R, system.r);
  host::put<D>(h.get(), TLSPH_FIELD_V, system.v);
  host::put<D>(h.get(), TLSPH_FIELD_A, system.a);
  host::put<D>(h.get(), TLSPH_FIELD_F, system.F);
  host::put<D>(h.get(), TLSPH_FIELD_DFDT, system.dFdt);
  host::put<D>(h.get(), TLSPH_FIELD_B0, system.B0);
  host::put(h.get(), TLSPH_FIELD_RHO, system.rho);
  put_external<D>(h.get(), system, external);
  const auto mat = host::to_dev(material);
  host::check(tlsph_dev_verlet_step(h.get(), &mat, dt));
  host::get<D>(h.get(), TLSPH_FIELD_R, system.r);
  host::get<D>(h.get(), TLSPH_FIELD_V, system.v);
  host::get<D>(h.get(), TLSPH_FIELD_A, system.a);
  host::get<D>(h.get(), TLSPH_FIELD_F, system.F);
  host::get<D>(h.get(), TLSPH_FIELD_DFDT, system.dFdt);
  host::get(h.get(), TLSPH_FIELD_RHO, system.rho);
}

template <int D>
StepSizes stable_dt(const ParticleSystem<D>& system, const Material& material, double h) {
  ReferenceNeighborhood<D> empty;
  empty.offsets.assign(system.size() + 1, 0);
  auto dev = host::upload<D>(system, empty, host::coarse_cutoff<D>(system, empty));
  host::put<D>(dev.get(), TLSPH_FIELD_V, system.v);
  host::put<D>(dev.get(), TLSPH_FIELD_A, system.a);
  const auto mat = host::to_dev(material);
  StepSizes s;
  host::check(tlsph_dev_stable_dt(dev.get(), &mat, h, &s.dt_acoustic));
  s.dt = s.dt_acoustic;
  return s;
}

template <int D>
double total_kinetic_energy(const ParticleSystem<D>& system) {
  ReferenceNeighborhood<D> empty;
  empty.offsets.assign(system.size() + 1, 0);
  auto dev = host::upload<D>(system, empty, host::coarse_cutoff<D>(system, empty));
  host::put<D>(dev.get(), TLSPH_FIELD_V, system.v);
  double e = 0.0;
  host::check(tlsph_dev_kinetic_energy(dev.get(), &e));
  return e;
}

// Diagnostic only (not on the hot path): host sum in the reference order.
template <int D>
double total_strain_energy(const ParticleSystem<D>& system, const Material& material) {
  double e = 0.0;
  for (std::size_t i = 0; i < system.size(); ++i) e += system.V0[i] * strain_energy_density<D>(system.F[i], material);
  return e;
}

#define TLSPH_INSTANTIATE(D)                                                                                      \
  template void compute_correction_matrices<D>(ParticleSystem<D>&, const ReferenceNeighborhood<D>&, int);         \
  template void compute_deformation_rate<D>(ParticleSystem<D>&, const ReferenceNeighborhood<D>&, int);            \
  template void update_density<D>(ParticleSystem<D>&, int);                                                       \
  template void compute_momentum_rhs<D>(ParticleSystem<D>&, const ReferenceNeighborhood<D>&, const Material&,     \
                                        const ExternalAccel<D>&, int);                                            \
  template void verlet_step<D>(ParticleSystem<D>&, const ReferenceNeighborhood<D>&, const Material&,              \
                               const ExternalAccel<D>&, double, int);                                             \
  template StepSizes stable_dt<D>(const ParticleSystem<D>&, const Material&, double);                             \
  template double total_kinetic_energy<D>(const ParticleSystem<D>&);                                              \
  template double total_strain_energy<D>(const ParticleSystem<D>&, const Material&);
TLSPH_INSTANTIATE(2)
TLSPH_INSTANTIATE(3)
#undef TLSPH_INSTANTIATE

}  // namespace tlsph
