// TL-SPH operators through the device (reference: proj/src/tlsph/integrator.cpp:12-188).
// Each operator runs on the device system kept resident for the caller's neighbourhood
// (resident.hpp) and moves only the ParticleSystem fields the reference operator reads (host ->
// device) and writes (device -> host), straight from and into the caller's vectors.
#include "tlsph/integrator.hpp"

#include <cmath>
#include <string>

#include "resident.hpp"
#include "tlsph/errors.hpp"

namespace tlsph {

namespace {

template <int D>
void put_external(tlsph_dev* dev, const ParticleSystem<D>& system, const ExternalAccel<D>& ext) {
  if (!ext.body.empty()) {
    require(ext.body.size() == system.size(), ErrorKind::InvalidArgument, "body force size mismatch");
    host::put(dev, TLSPH_FIELD_BODY, ext.body);
  } else {
    host::check(tlsph_dev_put(dev, TLSPH_FIELD_BODY, nullptr, TLSPH_LAYOUT_ROW_MAJOR));
  }
  double p[3] = {0, 0, 0}, nrm[3] = {0, 0, 0};
  double stiffness = 0.0;  // removes the plane
  if (ext.contact) {
    for (int d = 0; d < D; ++d) {
      p[d] = ext.contact->point[d];
      nrm[d] = ext.contact->normal[d];
    }
    stiffness = ext.contact->stiffness;
  }
  host::check(tlsph_dev_set_contact_plane(dev, p, nrm, stiffness));
}

// Per-particle constants the TL-SPH operators read (volumes, masses, densities, clamp flags).
template <int D>
void put_constants(tlsph_dev* dev, const ParticleSystem<D>& system) {
  host::refresh(dev, TLSPH_FIELD_V0, system.V0);
  host::refresh(dev, TLSPH_FIELD_M, system.m);
  host::put(dev, TLSPH_FIELD_RHO0, system.rho0);
  host::refresh(dev, TLSPH_FIELD_CONSTRAINED, system.constrained);
}

}  // namespace

// reads r0 (through the CSR), V0; writes B0 (integrator.cpp:12-42)
template <int D>
void compute_correction_matrices(ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh, int threads) {
  (void)threads;
  auto lease = host::resident<D>(system, nbh, nullptr);
  host::refresh(lease.get(), TLSPH_FIELD_V0, system.V0);
  host::check(tlsph_dev_correction_matrices(lease.get()));
  host::take(lease.get(), TLSPH_FIELD_B0, system.B0);
}

// reads v, B0, V0; writes dFdt (integrator.cpp:44-58)
template <int D>
void compute_deformation_rate(ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh, int threads) {
  (void)threads;
  auto lease = host::resident<D>(system, nbh, nullptr);
  host::refresh(lease.get(), TLSPH_FIELD_V0, system.V0);
  host::put(lease.get(), TLSPH_FIELD_V, system.v);
  host::put(lease.get(), TLSPH_FIELD_B0, system.B0);
  host::check(tlsph_dev_deformation_rate(lease.get()));
  host::take(lease.get(), TLSPH_FIELD_DFDT, system.dFdt);
}

// reads F, rho0; writes rho (integrator.cpp:60-78)
template <int D>
void update_density(ParticleSystem<D>& system, int threads) {
  (void)threads;
  auto lease = host::resident_any<D>(system);
  host::put(lease.get(), TLSPH_FIELD_F, system.F);
  host::put(lease.get(), TLSPH_FIELD_RHO0, system.rho0);
  host::put(lease.get(), TLSPH_FIELD_RHO, system.rho);
  const tlsph_status st = tlsph_dev_update_density(lease.get());
  const std::string msg = tlsph_dev_last_error();
  host::take(lease.get(), TLSPH_FIELD_RHO, system.rho);  // non-inverted particles are updated before the throw
  if (st == TLSPH_ERR_INVERTED_ELEMENT) throw Error(ErrorKind::InvertedElement, msg);
  host::check(st);
}

// reads F, B0, V0, m, r (contact), body; writes a (integrator.cpp:80-116)
template <int D>
void compute_momentum_rhs(ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh, const Material& material,
                          const ExternalAccel<D>& external, int threads) {
  (void)threads;
  auto lease = host::resident<D>(system, nbh, nullptr);
  put_constants<D>(lease.get(), system);
  host::put(lease.get(), TLSPH_FIELD_F, system.F);
  host::put(lease.get(), TLSPH_FIELD_B0, system.B0);
  host::put(lease.get(), TLSPH_FIELD_R, system.r);
  put_external<D>(lease.get(), system, external);
  const auto mat = host::to_dev(material);
  host::check(tlsph_dev_momentum_rhs(lease.get(), &mat));
  host::take(lease.get(), TLSPH_FIELD_A, system.a);
}

// reads r, v, F, dFdt, B0 and the constants, r0 (constraints), body; writes r, v, a, F, dFdt, rho
// (integrator.cpp:118-152)
template <int D>
void verlet_step(ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh, const Material& material,
                 const ExternalAccel<D>& external, double dt, int threads) {
  (void)threads;
  auto lease = host::resident<D>(system, nbh, nullptr);
  tlsph_dev* dev = lease.get();
  put_constants<D>(dev, system);
  host::refresh(dev, TLSPH_FIELD_R0, system.r0);
  host::put(dev, TLSPH_FIELD_R, system.r);
  host::put(dev, TLSPH_FIELD_V, system.v);
  host::put(dev, TLSPH_FIELD_F, system.F);
  host::put(dev, TLSPH_FIELD_DFDT, system.dFdt);
  host::put(dev, TLSPH_FIELD_B0, system.B0);
  put_external<D>(dev, system, external);
  const auto mat = host::to_dev(material);
  host::check(tlsph_dev_verlet_step(dev, &mat, dt));
  host::take(dev, TLSPH_FIELD_R, system.r);
  host::take(dev, TLSPH_FIELD_V, system.v);
  host::take(dev, TLSPH_FIELD_A, system.a);
  host::take(dev, TLSPH_FIELD_F, system.F);
  host::take(dev, TLSPH_FIELD_DFDT, system.dFdt);
  host::take(dev, TLSPH_FIELD_RHO, system.rho);
}

// reads v, a (integrator.cpp:154-169)
template <int D>
StepSizes stable_dt(const ParticleSystem<D>& system, const Material& material, double h) {
  auto lease = host::resident_any<D>(system);
  host::put(lease.get(), TLSPH_FIELD_V, system.v);
  host::put(lease.get(), TLSPH_FIELD_A, system.a);
  const auto mat = host::to_dev(material);
  StepSizes s;
  host::check(tlsph_dev_stable_dt(lease.get(), &mat, h, &s.dt_acoustic));
  s.dt = s.dt_acoustic;
  return s;
}

// reads v, m (integrator.cpp:171-178)
template <int D>
double total_kinetic_energy(const ParticleSystem<D>& system) {
  auto lease = host::resident_any<D>(system);
  host::put(lease.get(), TLSPH_FIELD_V, system.v);
  host::refresh(lease.get(), TLSPH_FIELD_M, system.m);
  double e = 0.0;
  host::check(tlsph_dev_kinetic_energy(lease.get(), &e));
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
