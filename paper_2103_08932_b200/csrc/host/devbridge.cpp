#include "devbridge.hpp"

#include <algorithm>
#include <stdexcept>

namespace tlsph::host {

void check(tlsph_status status) {
  if (status == TLSPH_OK) return;
  const std::string msg = tlsph_dev_last_error();
  switch (status) {
    case TLSPH_ERR_INVALID_ARGUMENT: throw Error(ErrorKind::InvalidArgument, msg);
    case TLSPH_ERR_PARSE: throw Error(ErrorKind::Parse, msg);
    case TLSPH_ERR_DEGENERATE_GEOMETRY: throw Error(ErrorKind::DegenerateGeometry, msg);
    case TLSPH_ERR_INVERTED_ELEMENT: throw Error(ErrorKind::InvertedElement, msg);
    case TLSPH_ERR_NUMERICAL_FAILURE: throw Error(ErrorKind::NumericalFailure, msg);
    case TLSPH_ERR_IO: throw Error(ErrorKind::Io, msg);
    default: throw std::runtime_error(msg);
  }
}

tlsph_dev_material to_dev(const Material& m) {
  tlsph_dev_material d{};
  d.model = m.model == ConstitutiveModel::NeoHookean ? 1 : 0;
  d.lambda = m.lambda;
  d.mu = m.mu;
  d.K = m.K;
  d.G = m.G;
  d.E = m.E;
  d.nu = m.nu;
  d.rho0 = m.rho0;
  d.c = m.c;
  return d;
}

template <int D>
double coarse_cutoff(const ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh) {
  // Operators that only walk the CSR do not depend on the grid; pick a cell
  // at least as large as the longest reference pair (so every CSR neighbour
  // lies in the 3^D stencil) and no finer than 1/256 of the body, which
  // bounds the cell count.
  double ext = 0.0;
  for (int d = 0; d < D; ++d) {
    double lo = system.r0[0][d], hi = lo;
    for (const auto& p : system.r0) {
      lo = std::min(lo, p[d]);
      hi = std::max(hi, p[d]);
    }
    ext = std::max(ext, hi - lo);
  }
  double mx = 0.0;
  for (double l : nbh.r0_len) mx = std::max(mx, l);
  const double c = std::max(mx * (1.0 + 1e-9), ext / 256.0);
  return c > 0.0 ? c : 1.0;
}

template double coarse_cutoff<2>(const ParticleSystem<2>&, const ReferenceNeighborhood<2>&);
template double coarse_cutoff<3>(const ParticleSystem<3>&, const ReferenceNeighborhood<3>&);

}  // namespace tlsph::host
