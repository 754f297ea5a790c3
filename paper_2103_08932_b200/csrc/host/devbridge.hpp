// Host <-> device bridge for the C++ operator API: every call crosses into
// the sm_100a kernels through the thin C ABI of include/tlsph/tlsph_dev.h.
#ifndef TLSPH_HOST_DEVBRIDGE_HPP
#define TLSPH_HOST_DEVBRIDGE_HPP

#include <string>
#include <vector>

#include "tlsph/errors.hpp"
#include "tlsph/material.hpp"
#include "tlsph/neighbors.hpp"
#include "tlsph/particle_system.hpp"
#include "tlsph/tlsph_dev.h"

namespace tlsph::host {

// Maps a device status to the reference's exception (InvalidArgument ... Io);
// TLSPH_ERR_INTERNAL (CUDA failures) becomes std::runtime_error.
void check(tlsph_status status);

class DevHandle {
 public:
  DevHandle() = default;
  explicit DevHandle(tlsph_dev* p) : p_(p) {}
  DevHandle(const DevHandle&) = delete;
  DevHandle& operator=(const DevHandle&) = delete;
  DevHandle(DevHandle&& o) noexcept : p_(o.p_) { o.p_ = nullptr; }
  DevHandle& operator=(DevHandle&& o) noexcept {
    if (this != &o) {
      reset();
      p_ = o.p_;
      o.p_ = nullptr;
    }
    return *this;
  }
  ~DevHandle() { reset(); }
  void reset() {
    if (p_) tlsph_dev_destroy(p_);
    p_ = nullptr;
  }
  tlsph_dev* get() const { return p_; }
  tlsph_dev** out() {
    reset();
    return &p_;
  }

 private:
  tlsph_dev* p_ = nullptr;
};

template <int D>
std::vector<double> flatten(const std::vector<Vec<D>>& a) {
  std::vector<double> out(a.size() * D);
  for (size_t i = 0; i < a.size(); ++i)
    for (int d = 0; d < D; ++d) out[i * D + d] = a[i][d];
  return out;
}

template <int D>
std::vector<double> flatten(const std::vector<Mat<D>>& a) {
  std::vector<double> out(a.size() * D * D);
  for (size_t i = 0; i < a.size(); ++i)
    for (int r = 0; r < D; ++r)
      for (int c = 0; c < D; ++c) out[(i * D + r) * D + c] = a[i](r, c);
  return out;
}

template <int D>
void unflatten(const std::vector<double>& in, std::vector<Vec<D>>& a) {
  for (size_t i = 0; i < a.size(); ++i)
    for (int d = 0; d < D; ++d) a[i][d] = in[i * D + d];
}

template <int D>
void unflatten(const std::vector<double>& in, std::vector<Mat<D>>& a) {
  for (size_t i = 0; i < a.size(); ++i)
    for (int r = 0; r < D; ++r)
      for (int c = 0; c < D; ++c) a[i](r, c) = in[(i * D + r) * D + c];
}

template <int D>
void put(tlsph_dev* dev, tlsph_dev_field f, const std::vector<Vec<D>>& a) {
  const auto flat = flatten<D>(a);
  check(tlsph_dev_set_field(dev, f, flat.data()));
}
template <int D>
void put(tlsph_dev* dev, tlsph_dev_field f, const std::vector<Mat<D>>& a) {
  const auto flat = flatten<D>(a);
  check(tlsph_dev_set_field(dev, f, flat.data()));
}
inline void put(tlsph_dev* dev, tlsph_dev_field f, const std::vector<double>& a) {
  check(tlsph_dev_set_field(dev, f, a.data()));
}
template <int D>
void get(tlsph_dev* dev, tlsph_dev_field f, std::vector<Vec<D>>& a) {
  std::vector<double> flat(a.size() * D);
  check(tlsph_dev_get_field(dev, f, flat.data()));
  unflatten<D>(flat, a);
}
template <int D>
void get(tlsph_dev* dev, tlsph_dev_field f, std::vector<Mat<D>>& a) {
  std::vector<double> flat(a.size() * D * D);
  check(tlsph_dev_get_field(dev, f, flat.data()));
  unflatten<D>(flat, a);
}
inline void get(tlsph_dev* dev, tlsph_dev_field f, std::vector<double>& a) {
  check(tlsph_dev_get_field(dev, f, a.data()));
}

tlsph_dev_material to_dev(const Material& m);

// A device system holding `system` and the caller's neighbourhood (reference
// order), with the cell grid for cutoff `cutoff`; ORDERED reductions so the
// operator API reproduces the reference arithmetic bit for bit.
template <int D>
DevHandle upload(const ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh, double cutoff);

// Grid cutoff for operators that never sweep: a single cell over the body.
template <int D>
double coarse_cutoff(const ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh);

}  // namespace tlsph::host

#endif  // TLSPH_HOST_DEVBRIDGE_HPP
