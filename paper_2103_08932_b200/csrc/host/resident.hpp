// Device-resident systems behind the C++ operator API.
//
// The reference's callers loop on operators over persistent host state (runner.cpp:341-391:
// stable_dt, verlet_step, strang_damping_sweep every step on one ParticleSystem and one
// ReferenceNeighborhood). The neighbourhood and the cell grid are fixed for a run, the particle
// fields change every call. So the drop-in keeps one device system per neighbourhood resident
// across calls -- the CSR (52 B per slot, ~1 GB at cfg2, ~30 GB at cfg4) crosses PCIe once --
// and each operator moves only the ParticleSystem fields the reference operator reads (host ->
// device) and writes (device -> host), straight from and into the caller's vectors.
//
// Keys. A neighbourhood is identified by the addresses and sizes of its six arrays plus a
// sampled content fingerprint (64 evenly spaced entries of each array), checked on every call;
// a cell grid by its geometry, the address of cell_of and a sampled fingerprint of it, verified
// once against the device's own binning. build_reference_neighborhoods registers the device
// system it built the CSR with, so a reference caller never uploads the CSR at all.
// Per-particle inputs are uploaded on every call; the ones derived data depends on (m,
// constrained, V0, r0) go through tlsph_dev_refresh, which rebuilds that data only when the
// caller really changed them. Editing a neighbourhood's arrays in place so that no sampled
// entry changes is not detected: build a new neighbourhood, or call release_resident().
#ifndef TLSPH_HOST_RESIDENT_HPP
#define TLSPH_HOST_RESIDENT_HPP

#include <cstdint>
#include <memory>
#include <mutex>

#include "devbridge.hpp"
#include "tlsph/neighbors.hpp"
#include "tlsph/particle_system.hpp"

namespace tlsph::host {

struct CsrIdentity {
  int dim = 0;
  std::size_t n = 0;
  std::int64_t slots = 0;
  const void* ptr[6] = {};
  std::uint64_t fingerprint = 0;
  bool operator==(const CsrIdentity& o) const;
};

struct GridIdentity {
  double cell = 0.0;
  double origin[3] = {0, 0, 0};
  int dims[3] = {1, 1, 1};
  const void* cell_of = nullptr;
  std::size_t ncells = 0;
  std::uint64_t fingerprint = 0;
  bool operator==(const GridIdentity& o) const;
};

template <int D>
CsrIdentity identify(const ReferenceNeighborhood<D>& nbh);
template <int D>
GridIdentity identify(const CellGrid<D>& grid);

struct ResidentEntry;

// Exclusive use of one resident device system for the duration of an operator call.
class Lease {
 public:
  Lease(std::shared_ptr<ResidentEntry> e);
  Lease(Lease&&) noexcept = default;
  ~Lease();
  tlsph_dev* get() const;

 private:
  std::shared_ptr<ResidentEntry> e_;
  std::unique_lock<std::mutex> lock_;
};

// The device system holding `nbh` (and sweeping with `grid` when given), built on a miss.
template <int D>
Lease resident(const ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh, const CellGrid<D>* grid);
// Any resident system of `system`'s size, for the CSR-free operators (stable_dt, kinetic energy,
// update_density); a neighbourhood-free one is built on a miss.
template <int D>
Lease resident_any(const ParticleSystem<D>& system);
// Registers a device system whose CSR `nbh` was just copied out of (build_reference_neighborhoods).
template <int D>
void adopt(DevHandle&& h, const ReferenceNeighborhood<D>& nbh);
// Drops every resident system (frees their device memory).
void release_resident();

// Applies the operator-API reduction mode (tlsph/device.hpp) to a leased system.
void apply_mode(tlsph_dev* dev);

// Field transfers in the caller's storage (no repacking): ParticleSystem vectors of Vec<D>,
// Mat<D> (column-major records) or doubles; constrained as bytes.
template <typename T>
void put(tlsph_dev* dev, tlsph_dev_field f, const std::vector<T>& a) {
  constexpr int layout = T::Cols > 1 ? TLSPH_LAYOUT_COL_MAJOR : TLSPH_LAYOUT_ROW_MAJOR;
  check(tlsph_dev_put(dev, f, a.data(), layout));
}
inline void put(tlsph_dev* dev, tlsph_dev_field f, const std::vector<double>& a) {
  check(tlsph_dev_put(dev, f, a.data(), TLSPH_LAYOUT_ROW_MAJOR));
}
template <typename T>
void refresh(tlsph_dev* dev, tlsph_dev_field f, const std::vector<T>& a) {
  constexpr int layout = T::Cols > 1 ? TLSPH_LAYOUT_COL_MAJOR : TLSPH_LAYOUT_ROW_MAJOR;
  int changed = 0;
  check(tlsph_dev_refresh(dev, f, a.data(), layout, &changed));
}
inline void refresh(tlsph_dev* dev, tlsph_dev_field f, const std::vector<double>& a) {
  int changed = 0;
  check(tlsph_dev_refresh(dev, f, a.data(), TLSPH_LAYOUT_ROW_MAJOR, &changed));
}
inline void refresh(tlsph_dev* dev, tlsph_dev_field f, const std::vector<std::uint8_t>& a) {
  int changed = 0;
  check(tlsph_dev_refresh(dev, f, a.data(), TLSPH_LAYOUT_ROW_MAJOR, &changed));
}
template <typename T>
void take(tlsph_dev* dev, tlsph_dev_field f, std::vector<T>& a) {
  constexpr int layout = T::Cols > 1 ? TLSPH_LAYOUT_COL_MAJOR : TLSPH_LAYOUT_ROW_MAJOR;
  check(tlsph_dev_take(dev, f, a.data(), layout));
}
inline void take(tlsph_dev* dev, tlsph_dev_field f, std::vector<double>& a) {
  check(tlsph_dev_take(dev, f, a.data(), TLSPH_LAYOUT_ROW_MAJOR));
}

}  // namespace tlsph::host

#endif  // TLSPH_HOST_RESIDENT_HPP
