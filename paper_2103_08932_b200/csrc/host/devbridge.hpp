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

tlsph_dev_material to_dev(const Material& m);

// Grid cutoff for operators that never sweep: a single cell over the body.
template <int D>
double coarse_cutoff(const ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh);

}  // namespace tlsph::host

#endif  // TLSPH_HOST_DEVBRIDGE_HPP
