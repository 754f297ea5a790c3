// Device-resident systems behind the C++ operator API (see resident.hpp).
#include "resident.hpp"

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <list>

#include "tlsph/device.hpp"
#include "tlsph/errors.hpp"

namespace tlsph {

namespace {
std::atomic<int> g_reduction{static_cast<int>(Reduction::Ordered)};
}

void set_operator_reduction(Reduction mode) { g_reduction.store(static_cast<int>(mode)); }
Reduction operator_reduction() { return static_cast<Reduction>(g_reduction.load()); }
void release_device_state() { host::release_resident(); }

namespace {
template <typename V>
void pin_vector(V& v, bool on) {
  if (v.empty()) return;
  if (on) host::check(tlsph_dev_host_register(v.data(), v.size() * sizeof(v[0])));
  else host::check(tlsph_dev_host_unregister(v.data()));
}
template <int D>
void pin_all(ParticleSystem<D>& s, std::vector<Vec<D>>* body, bool on) {
  pin_vector(s.r0, on);
  pin_vector(s.r, on);
  pin_vector(s.v, on);
  pin_vector(s.a, on);
  pin_vector(s.F, on);
  pin_vector(s.dFdt, on);
  pin_vector(s.B0, on);
  pin_vector(s.V0, on);
  pin_vector(s.m, on);
  pin_vector(s.rho0, on);
  pin_vector(s.rho, on);
  pin_vector(s.constrained, on);
  if (body) pin_vector(*body, on);
}
}  // namespace

template <int D>
void pin_host_memory(ParticleSystem<D>& system, std::vector<Vec<D>>* body) {
  pin_all<D>(system, body, true);
}
template <int D>
void unpin_host_memory(ParticleSystem<D>& system, std::vector<Vec<D>>* body) {
  pin_all<D>(system, body, false);
}
template void pin_host_memory<2>(ParticleSystem<2>&, std::vector<Vec<2>>*);
template void pin_host_memory<3>(ParticleSystem<3>&, std::vector<Vec<3>>*);
template void unpin_host_memory<2>(ParticleSystem<2>&, std::vector<Vec<2>>*);
template void unpin_host_memory<3>(ParticleSystem<3>&, std::vector<Vec<3>>*);

namespace host {

static_assert(sizeof(Vec<3>) == 3 * sizeof(double) && sizeof(Mat<3>) == 9 * sizeof(double),
              "ParticleSystem records must be plain doubles for zero-copy transfers");
static_assert(sizeof(Vec<2>) == 2 * sizeof(double) && sizeof(Mat<2>) == 4 * sizeof(double),
              "ParticleSystem records must be plain doubles for zero-copy transfers");

namespace {

constexpr int kSamples = 64;

std::uint64_t mix(std::uint64_t h, std::uint64_t x) {
  h ^= x + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  return h;
}

// 64 evenly spaced entries (first and last included) of an array of `count` records of `bytes`.
std::uint64_t sample(std::uint64_t h, const void* data, std::size_t count, std::size_t bytes) {
  h = mix(h, count);
  if (count == 0) return h;
  const auto* p = static_cast<const unsigned char*>(data);
  const int k = static_cast<int>(std::min<std::size_t>(count, kSamples));
  for (int s = 0; s < k; ++s) {
    const std::size_t i = k == 1 ? 0 : (count - 1) * static_cast<std::size_t>(s) / static_cast<std::size_t>(k - 1);
    for (std::size_t b = 0; b < bytes; b += sizeof(std::uint64_t)) {
      std::uint64_t w = 0;
      std::memcpy(&w, p + i * bytes + b, std::min(sizeof(w), bytes - b));
      h = mix(h, w);
    }
  }
  return h;
}

}  // namespace

bool CsrIdentity::operator==(const CsrIdentity& o) const {
  return dim == o.dim && n == o.n && slots == o.slots && std::equal(ptr, ptr + 6, o.ptr) &&
         fingerprint == o.fingerprint;
}

bool GridIdentity::operator==(const GridIdentity& o) const {
  return cell == o.cell && std::equal(origin, origin + 3, o.origin) && std::equal(dims, dims + 3, o.dims) &&
         cell_of == o.cell_of && ncells == o.ncells && fingerprint == o.fingerprint;
}

template <int D>
CsrIdentity identify(const ReferenceNeighborhood<D>& nbh) {
  CsrIdentity id;
  id.dim = D;
  id.n = nbh.particle_count();
  id.slots = nbh.offsets.empty() ? 0 : nbh.offsets.back();
  const void* p[6] = {nbh.offsets.data(), nbh.neighbor.data(), nbh.r0_len.data(),
                      nbh.e0.data(),      nbh.dwdr0.data(),    nbh.pair_factor.data()};
  std::copy(p, p + 6, id.ptr);
  std::uint64_t h = 0;
  h = sample(h, nbh.offsets.data(), nbh.offsets.size(), sizeof(std::int64_t));
  h = sample(h, nbh.neighbor.data(), nbh.neighbor.size(), sizeof(int));
  h = sample(h, nbh.r0_len.data(), nbh.r0_len.size(), sizeof(double));
  h = sample(h, nbh.e0.data(), nbh.e0.size(), sizeof(Vec<D>));
  h = sample(h, nbh.dwdr0.data(), nbh.dwdr0.size(), sizeof(double));
  h = sample(h, nbh.pair_factor.data(), nbh.pair_factor.size(), sizeof(double));
  id.fingerprint = h;
  return id;
}

template <int D>
GridIdentity identify(const CellGrid<D>& grid) {
  GridIdentity id;
  id.cell = grid.cell_size;
  for (int d = 0; d < D; ++d) {
    id.origin[d] = grid.origin[d];
    id.dims[d] = grid.dims[d];
  }
  id.cell_of = grid.cell_of.data();
  id.ncells = grid.cells.size();
  id.fingerprint = sample(0, grid.cell_of.data(), grid.cell_of.size(), sizeof(int));
  return id;
}

struct ResidentEntry {
  CsrIdentity csr;
  bool csr_free = false;       // built without a neighbourhood (CSR-free operators only)
  GridIdentity grid;           // a caller grid verified against the device binning
  bool grid_verified = false;
  DevHandle h;
  std::mutex use;
};

namespace {

class Registry {
 public:
  static Registry& get() {
    static Registry r;
    return r;
  }

  std::shared_ptr<ResidentEntry> find(const CsrIdentity& id) {
    std::lock_guard<std::mutex> g(mu_);
    for (auto it = entries_.begin(); it != entries_.end(); ++it)
      if (!(*it)->csr_free && (*it)->csr == id) {
        entries_.splice(entries_.begin(), entries_, it);  // most recently used first
        return entries_.front();
      }
    return nullptr;
  }

  std::shared_ptr<ResidentEntry> find_size(int dim, std::size_t n) {
    std::lock_guard<std::mutex> g(mu_);
    for (auto it = entries_.begin(); it != entries_.end(); ++it)
      if ((*it)->csr.dim == dim && (*it)->csr.n == n) {
        entries_.splice(entries_.begin(), entries_, it);
        return entries_.front();
      }
    return nullptr;
  }

  void insert(std::shared_ptr<ResidentEntry> e) {
    std::lock_guard<std::mutex> g(mu_);
    for (auto it = entries_.begin(); it != entries_.end();)  // one entry per neighbourhood storage
      if (!(*it)->csr_free && !e->csr_free && std::equal(e->csr.ptr, e->csr.ptr + 6, (*it)->csr.ptr))
        it = entries_.erase(it);
      else
        ++it;
    entries_.push_front(std::move(e));
    while (entries_.size() > capacity()) entries_.pop_back();  // a leased entry lives on in its lease
  }

  void clear() {
    std::lock_guard<std::mutex> g(mu_);
    entries_.clear();
  }

 private:
  static std::size_t capacity() {
    const char* e = std::getenv("TLSPH_RESIDENT_SYSTEMS");
    const long v = e ? std::strtol(e, nullptr, 10) : 2;
    return static_cast<std::size_t>(std::max(1L, v));
  }
  std::mutex mu_;
  std::list<std::shared_ptr<ResidentEntry>> entries_;
};

template <int D>
void flat_positions(const std::vector<Vec<D>>& r0, std::vector<double>& out) {
  out.resize(r0.size() * D);
  std::memcpy(out.data(), r0.data(), out.size() * sizeof(double));
}

// A device system holding the caller's CSR, binned with cell size `cutoff`.
template <int D>
std::shared_ptr<ResidentEntry> build(const ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh,
                                     double cutoff) {
  const std::size_t n = system.size();
  require(n > 0, ErrorKind::InvalidArgument, "particle system is empty");
  require(nbh.offsets.size() == n + 1, ErrorKind::InvalidArgument, "neighbourhood does not match the system");
  auto e = std::make_shared<ResidentEntry>();
  e->csr = identify<D>(nbh);
  static_assert(sizeof(Vec<D>) == D * sizeof(double));
  check(tlsph_dev_create_with_csr(D, n, reinterpret_cast<const double*>(system.r0.data()), system.V0.data(),
                                  system.rho0.data(), system.constrained.data(), 0.5 * cutoff, nbh.offsets.data(),
                                  nbh.neighbor.data(), nbh.r0_len.data(),
                                  reinterpret_cast<const double*>(nbh.e0.data()), nbh.dwdr0.data(),
                                  nbh.pair_factor.data(), e->h.out()));
  return e;
}

// Checks a caller grid against the device binning (cell size, origin, dims, every cell_of).
template <int D>
bool grid_matches(tlsph_dev* dev, const CellGrid<D>& grid) {
  int dims[3] = {1, 1, 1};
  double origin[3] = {0, 0, 0}, cell = 0.0;
  std::int64_t ncells = 0;
  check(tlsph_dev_grid_info(dev, dims, origin, &cell, &ncells));
  if (cell != grid.cell_size || static_cast<std::size_t>(ncells) != grid.cells.size()) return false;
  for (int d = 0; d < D; ++d)
    if (dims[d] != grid.dims[d] || origin[d] != grid.origin[d]) return false;
  std::vector<std::int32_t> cell_of(grid.cell_of.size());
  check(tlsph_dev_grid_cells(dev, cell_of.data(), nullptr, nullptr));
  return std::equal(cell_of.begin(), cell_of.end(), grid.cell_of.begin());
}

}  // namespace

Lease::Lease(std::shared_ptr<ResidentEntry> e) : e_(std::move(e)), lock_(e_->use) {}
Lease::~Lease() = default;
tlsph_dev* Lease::get() const { return e_->h.get(); }

void apply_mode(tlsph_dev* dev) {
  check(tlsph_dev_set_reduction(dev, operator_reduction() == Reduction::Fast ? TLSPH_REDUCTION_FAST
                                                                             : TLSPH_REDUCTION_ORDERED));
}

template <int D>
Lease resident(const ParticleSystem<D>& system, const ReferenceNeighborhood<D>& nbh, const CellGrid<D>* grid) {
  const CsrIdentity id = identify<D>(nbh);
  require(id.n == system.size(), ErrorKind::InvalidArgument, "neighbourhood does not match the system");
  std::shared_ptr<ResidentEntry> e = Registry::get().find(id);
  if (e && grid) {
    const GridIdentity gid = identify<D>(*grid);
    if (!(e->grid_verified && e->grid == gid)) {
      Lease l(e);
      if (grid_matches<D>(l.get(), *grid)) {
        e->grid = gid;
        e->grid_verified = true;
      } else {
        e = nullptr;  // rebuilt below with the caller's cell size
      }
    }
  }
  if (!e) {
    const double cutoff = grid ? grid->cell_size : coarse_cutoff<D>(system, nbh);
    e = build<D>(system, nbh, cutoff);
    if (grid) {
      require(grid_matches<D>(e->h.get(), *grid), ErrorKind::InvalidArgument,
              "the cell grid is not build_cell_grid of the reference positions with its cell size");
      e->grid = identify<D>(*grid);
      e->grid_verified = true;
    }
    Registry::get().insert(e);
  }
  Lease l(std::move(e));
  apply_mode(l.get());
  return l;
}

template <int D>
Lease resident_any(const ParticleSystem<D>& system) {
  const std::size_t n = system.size();
  require(n > 0, ErrorKind::InvalidArgument, "particle system is empty");
  std::shared_ptr<ResidentEntry> e = Registry::get().find_size(D, n);
  if (!e) {
    ReferenceNeighborhood<D> empty;
    empty.offsets.assign(n + 1, 0);
    e = build<D>(system, empty, coarse_cutoff<D>(system, empty));
    e->csr_free = true;
    e->csr.ptr[0] = nullptr;
    Registry::get().insert(e);
  }
  Lease l(std::move(e));
  apply_mode(l.get());
  return l;
}

template <int D>
void adopt(DevHandle&& h, const ReferenceNeighborhood<D>& nbh) {
  auto e = std::make_shared<ResidentEntry>();
  e->csr = identify<D>(nbh);
  e->h = std::move(h);
  Registry::get().insert(std::move(e));
}

void release_resident() { Registry::get().clear(); }

template CsrIdentity identify<2>(const ReferenceNeighborhood<2>&);
template CsrIdentity identify<3>(const ReferenceNeighborhood<3>&);
template GridIdentity identify<2>(const CellGrid<2>&);
template GridIdentity identify<3>(const CellGrid<3>&);
template Lease resident<2>(const ParticleSystem<2>&, const ReferenceNeighborhood<2>&, const CellGrid<2>*);
template Lease resident<3>(const ParticleSystem<3>&, const ReferenceNeighborhood<3>&, const CellGrid<3>*);
template Lease resident_any<2>(const ParticleSystem<2>&);
template Lease resident_any<3>(const ParticleSystem<3>&);
template void adopt<2>(DevHandle&&, const ReferenceNeighborhood<2>&);
template void adopt<3>(DevHandle&&, const ReferenceNeighborhood<3>&);

}  // namespace host
}  // namespace tlsph
