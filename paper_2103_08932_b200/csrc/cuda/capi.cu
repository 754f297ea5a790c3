#include <atomic>
// extern "C" boundary of libtlsph_cuda.so (declared in include/tlsph/tlsph_dev.h).
// Exception-free: every entry point maps DevError / std::exception to a
// tlsph_status and a thread-local message, as the reference C API does
// (proj/src/capi.cpp:12,26-42).
#include <cstring>
#include <memory>
#include <random>
#include <string>

#include "system.cuh"

using tlsph_cuda::DevError;
using tlsph_cuda::DevSystem;
using tlsph_cuda::IpcExport;

namespace {

thread_local std::string g_dev_err;
int g_default_device = 0;

template <typename Fn>
tlsph_status guarded(Fn&& fn) {
  try {
    fn();
    g_dev_err.clear();
    return TLSPH_OK;
  } catch (const DevError& e) {
    g_dev_err = e.what();
    return e.status;
  } catch (const std::exception& e) {
    g_dev_err = e.what();
    return TLSPH_ERR_INTERNAL;
  } catch (...) {
    g_dev_err = "unknown error";
    return TLSPH_ERR_INTERNAL;
  }
}

DevSystem& sys(tlsph_dev* d) {
  if (!d) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "device handle must not be null");
  CK(cudaSetDevice(d->sys.device));
  return d->sys;
}
const DevSystem& sys(const tlsph_dev* d) {
  if (!d) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "device handle must not be null");
  CK(cudaSetDevice(d->sys.device));
  return d->sys;
}

std::unique_ptr<tlsph_dev> new_handle() {
  auto d = std::make_unique<tlsph_dev>();
  d->sys.device = g_default_device;
  CK(cudaSetDevice(d->sys.device));
  return d;
}

void require_material(const tlsph_dev_material* m) {
  if (!m) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "material must not be null");
}

}  // namespace

extern "C" {

const char* tlsph_dev_last_error(void) { return g_dev_err.c_str(); }

int tlsph_dev_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

tlsph_status tlsph_dev_select_device(int ordinal) {
  return guarded([&] {
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    if (ordinal < 0 || ordinal >= count)
      throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "device ordinal " + std::to_string(ordinal) + " out of range");
    g_default_device = ordinal;
  });
}

tlsph_status tlsph_dev_create(int dim, size_t n, const double* r0, const double* V0, const double* rho0,
                              const uint8_t* constrained, double h, tlsph_dev** out) {
  if (!out) {
    g_dev_err = "out must not be null";
    return TLSPH_ERR_INVALID_ARGUMENT;
  }
  *out = nullptr;
  return guarded([&] {
    auto d = new_handle();
    d->sys.init_common(dim, n, r0, V0, rho0, constrained, h);
    d->sys.build_neighbourhoods();
    *out = d.release();
  });
}

tlsph_status tlsph_dev_create_with_csr(int dim, size_t n, const double* r0, const double* V0, const double* rho0,
                                       const uint8_t* constrained, double h, const int64_t* offsets,
                                       const int32_t* neighbor, const double* r0_len, const double* e0,
                                       const double* dwdr0, const double* pair_factor, tlsph_dev** out) {
  if (!out) {
    g_dev_err = "out must not be null";
    return TLSPH_ERR_INVALID_ARGUMENT;
  }
  *out = nullptr;
  return guarded([&] {
    if (!offsets) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "offsets must not be null");
    auto d = new_handle();
    d->sys.init_common(dim, n, r0, V0, rho0, constrained, h);
    d->sys.load_csr(offsets, neighbor, r0_len, e0, dwdr0, pair_factor);
    *out = d.release();
  });
}

tlsph_status tlsph_dev_create_grid(int dim, size_t n, const double* positions, double cutoff, tlsph_dev** out) {
  if (!out) {
    g_dev_err = "out must not be null";
    return TLSPH_ERR_INVALID_ARGUMENT;
  }
  *out = nullptr;
  return guarded([&] {
    if (!(cutoff > 0.0)) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "cell grid cutoff must be positive");
    if (n == 0) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "cell grid needs at least one particle");
    const std::vector<double> ones(n, 1.0);
    auto d = new_handle();
    d->sys.init_common(dim, n, positions, ones.data(), ones.data(), nullptr, 0.5 * cutoff);
    *out = d.release();
  });
}

tlsph_status tlsph_dev_create_in_grid(int dim, size_t n, const double* r0, const double* V0, const double* rho0,
                                      const uint8_t* constrained, double h, const double* origin, const int* dims,
                                      tlsph_dev** out) {
  if (!out) {
    g_dev_err = "out must not be null";
    return TLSPH_ERR_INVALID_ARGUMENT;
  }
  *out = nullptr;
  return guarded([&] {
    if (!origin || !dims) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "origin and dims must not be null");
    auto d = new_handle();
    d->sys.grid_given = true;
    for (int k = 0; k < dim && k < 3; ++k) {
      d->sys.given_origin[k] = origin[k];
      d->sys.given_dims[k] = dims[k];
    }
    d->sys.init_common(dim, n, r0, V0, rho0, constrained, h);
    d->sys.build_neighbourhoods();
    *out = d.release();
  });
}

tlsph_status tlsph_dev_set_task_range(tlsph_dev* dev, int x0, int x1) {
  return guarded([&] {
    DevSystem& s = sys(dev);
    if (x0 < 0 || x1 > s.dims[0] || x0 >= x1)
      throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "task range must satisfy 0 <= x0 < x1 <= dims[0]");
    s.task_x0 = x0;
    s.task_x1 = x1;
    s.build_colour_lists();
    s.build_own_mask();
  });
}

tlsph_status tlsph_dev_damping_phase(tlsph_dev* dev, tlsph_dev_scheme scheme, double eta_tilde, double dt, int pass,
                                     int index) {
  return guarded([&] {
    DevSystem& s = sys(dev);
    if (eta_tilde == 0.0) return;  // damping.cpp:132
    if (scheme != TLSPH_SCHEME_PARTICLE_SPLIT && scheme != TLSPH_SCHEME_PAIRWISE_SPLIT)
      throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "only the split schemes are swept");
    s.enqueue_sweep_phase(scheme, eta_tilde, dt, pass, index);
    s.sync();
  });
}

tlsph_status tlsph_dev_sweep_linked(tlsph_dev* const* slabs, int nslabs, tlsph_dev_scheme scheme, double eta_tilde,
                                    double dt, int count) {
  return guarded([&] {
    if (!slabs || nslabs < 1) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "no slabs");
    if (count < 0) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "negative sweep count");
    if (scheme != TLSPH_SCHEME_PARTICLE_SPLIT && scheme != TLSPH_SCHEME_PAIRWISE_SPLIT)
      throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "only the split schemes are swept");
    std::vector<DevSystem*> sl;
    for (int r = 0; r < nslabs; ++r) {
      if (!slabs[r]) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "null slab");
      sl.push_back(&sys(slabs[r]));
    }
    if (eta_tilde == 0.0 || count == 0) return;  // damping.cpp:132
    sweep_linked(sl, scheme, eta_tilde, dt, count);
  });
}

size_t tlsph_dev_ipc_size(void) { return sizeof(IpcExport); }

tlsph_status tlsph_dev_ipc_export(tlsph_dev* dev, void* blob) {
  return guarded([&] {
    if (!blob) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "null blob");
    IpcExport e;
    sys(dev).ipc_export(&e);
    std::memcpy(blob, &e, sizeof(e));
  });
}

tlsph_status tlsph_dev_link_peer_ipc(tlsph_dev* dev, int side, const void* peer_blob, const int64_t* peer_cell_start) {
  return guarded([&] {
    if (!peer_blob || !peer_cell_start) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "null peer export");
    IpcExport e;
    std::memcpy(&e, peer_blob, sizeof(e));
    static_assert(sizeof(int64_t) == sizeof(long long), "cell table");
    sys(dev).link_peer_ipc(side, e, reinterpret_cast<const long long*>(peer_cell_start));
  });
}

tlsph_status tlsph_dev_sweep_phase_ipc(tlsph_dev* dev, tlsph_dev_scheme scheme, double eta_tilde, double dt, int q,
                                       int wait_q) {
  return guarded([&] {
    if (scheme != TLSPH_SCHEME_PARTICLE_SPLIT && scheme != TLSPH_SCHEME_PAIRWISE_SPLIT)
      throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "only the split schemes are swept");
    sys(dev).sweep_phase_ipc(scheme, eta_tilde, dt, q, wait_q);
  });
}

tlsph_status tlsph_dev_push_halo_ipc(tlsph_dev* dev, tlsph_dev_column_field field) {
  return guarded([&] { sys(dev).push_halo_ipc(field); });
}

tlsph_status tlsph_dev_wait_halo_ipc(tlsph_dev* dev, tlsph_dev_column_field field) {
  return guarded([&] { sys(dev).wait_halo_ipc(field); });
}

tlsph_status tlsph_dev_mark_ipc(tlsph_dev* dev) {
  return guarded([&] { sys(dev).mark_ipc(); });
}

tlsph_status tlsph_dev_wait_mark_ipc(tlsph_dev* dev) {
  return guarded([&] { sys(dev).wait_mark_ipc(); });
}

tlsph_status tlsph_dev_wait_phase_ipc(tlsph_dev* dev, int q) {
  return guarded([&] { sys(dev).wait_phase_ipc(q); });
}

tlsph_status tlsph_dev_synchronize(tlsph_dev* dev) {
  return guarded([&] {
    DevSystem& s = sys(dev);
    CK(cudaSetDevice(s.device));
    s.sync();
  });
}

tlsph_status tlsph_dev_timer_start(tlsph_dev* dev) {
  return guarded([&] {
    DevSystem& s = sys(dev);
    CK(cudaSetDevice(s.device));
    for (cudaEvent_t& e : s.timer_ev)
      if (!e) CK(cudaEventCreate(&e));
    CK(cudaEventRecord(s.timer_ev[0], s.stream));
  });
}

double tlsph_dev_timer_stop(tlsph_dev* dev) {
  double out = -1.0;
  const tlsph_status st = guarded([&] {
    DevSystem& s = sys(dev);
    if (!s.timer_ev[0]) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "timer not started");
    CK(cudaSetDevice(s.device));
    CK(cudaEventRecord(s.timer_ev[1], s.stream));
    CK(cudaEventSynchronize(s.timer_ev[1]));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, s.timer_ev[0], s.timer_ev[1]));
    out = ms * 1e-3;
  });
  return st == TLSPH_OK ? out : -1.0;
}

tlsph_status tlsph_dev_link_peer(tlsph_dev* dev, int side, tlsph_dev* peer) {
  return guarded([&] {
    if (!peer) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "peer must not be null");
    DevSystem& s = sys(dev);
    DevSystem& p = sys(peer);
    if (s.device != p.device) {  // NVLink peer access for the fused stores
      int ok = 0;
      CK(cudaDeviceCanAccessPeer(&ok, s.device, p.device));
      if (!ok) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "peer device is not reachable by peer access");
      CK(cudaSetDevice(s.device));
      const cudaError_t e = cudaDeviceEnablePeerAccess(p.device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
      cudaGetLastError();
    }
    s.link_peer(side, p);
  });
}

int64_t tlsph_dev_column_count(const tlsph_dev* dev, int x) {
  int64_t c = -1;
  const tlsph_status st = guarded([&] { c = sys(dev).column_count(x); });
  return st == TLSPH_OK ? c : -1;
}

tlsph_status tlsph_dev_pack_column(tlsph_dev* dev, int x, double* device_dst) {
  return guarded([&] { sys(dev).pack_column(TLSPH_DEV_COLUMN_VELOCITY, x, device_dst); });
}

tlsph_status tlsph_dev_unpack_column(tlsph_dev* dev, int x, const double* device_src) {
  return guarded([&] { sys(dev).unpack_column(TLSPH_DEV_COLUMN_VELOCITY, x, device_src); });
}

int tlsph_dev_column_width(const tlsph_dev* dev, tlsph_dev_column_field field) {
  int w = -1;
  const tlsph_status st = guarded([&] { w = sys(dev).column_width(field); });
  return st == TLSPH_OK ? w : -1;
}

tlsph_status tlsph_dev_pack_column_field(tlsph_dev* dev, tlsph_dev_column_field field, int x, double* device_dst) {
  return guarded([&] { sys(dev).pack_column(field, x, device_dst); });
}

tlsph_status tlsph_dev_unpack_column_field(tlsph_dev* dev, tlsph_dev_column_field field, int x,
                                           const double* device_src) {
  return guarded([&] { sys(dev).unpack_column(field, x, device_src); });
}

tlsph_status tlsph_dev_set_contact_plane(tlsph_dev* dev, const double* point, const double* normal,
                                         double stiffness) {
  return guarded([&] {
    DevSystem& s = sys(dev);
    if (!(stiffness > 0.0)) {
      s.contact = false;
      return;
    }
    if (!point || !normal) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "point and normal must not be null");
    for (int d = 0; d < 3; ++d) {
      s.cp_point[d] = d < s.D ? point[d] : 0.0;
      s.cp_normal[d] = d < s.D ? normal[d] : 0.0;
    }
    s.cp_k = stiffness;
    s.contact = true;
  });
}

void tlsph_dev_destroy(tlsph_dev* dev) { delete dev; }

size_t tlsph_dev_size(const tlsph_dev* dev) { return dev ? static_cast<size_t>(dev->sys.n) : 0; }
int tlsph_dev_dim(const tlsph_dev* dev) { return dev ? dev->sys.D : 0; }
int64_t tlsph_dev_slot_count(const tlsph_dev* dev) { return dev ? dev->sys.nslots : 0; }

tlsph_status tlsph_dev_set_field(tlsph_dev* dev, tlsph_dev_field field, const double* host) {
  return guarded([&] { sys(dev).set_field(field, host); });
}

tlsph_status tlsph_dev_put(tlsph_dev* dev, tlsph_dev_field field, const void* host, int layout) {
  return guarded([&] { sys(dev).put_record(field, host, layout, false, nullptr); });
}

tlsph_status tlsph_dev_refresh(tlsph_dev* dev, tlsph_dev_field field, const void* host, int layout, int* changed) {
  return guarded([&] { sys(dev).put_record(field, host, layout, true, changed); });
}

tlsph_status tlsph_dev_host_register(void* host, size_t bytes) {
  return guarded([&] {
    if (!host || bytes == 0) return;
    const cudaError_t e = cudaHostRegister(host, bytes, cudaHostRegisterDefault);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {
      cudaGetLastError();
      return;
    }
    CK(e);
  });
}

tlsph_status tlsph_dev_host_unregister(void* host) {
  return guarded([&] {
    if (!host) return;
    const cudaError_t e = cudaHostUnregister(host);
    if (e == cudaErrorHostMemoryNotRegistered) {
      cudaGetLastError();
      return;
    }
    CK(e);
  });
}

void tlsph_dev_transfer_bytes(uint64_t* h2d, uint64_t* d2h) {
  if (h2d) *h2d = tlsph_cuda::g_h2d_bytes.load();
  if (d2h) *d2h = tlsph_cuda::g_d2h_bytes.load();
}

tlsph_status tlsph_dev_take(const tlsph_dev* dev, tlsph_dev_field field, void* host, int layout) {
  return guarded([&] { sys(dev).take_record(field, host, layout); });
}

tlsph_status tlsph_dev_get_field(const tlsph_dev* dev, tlsph_dev_field field, double* host) {
  return guarded([&] { sys(dev).get_field(field, host); });
}

tlsph_status tlsph_dev_set_reduction(tlsph_dev* dev, tlsph_dev_reduction mode) {
  return guarded([&] {
    if (mode != TLSPH_REDUCTION_FAST && mode != TLSPH_REDUCTION_ORDERED)
      throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "unknown reduction mode");
    sys(dev).reduction = mode;
  });
}

tlsph_status tlsph_dev_set_resort(tlsph_dev* dev, int on) {
  return guarded([&] { sys(dev).set_resort(on != 0); });
}

tlsph_status tlsph_dev_current_cells(const tlsph_dev* dev, int64_t* cell_start, int32_t* order) {
  return guarded([&] {
    if (!cell_start || !order) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "null output array");
    sys(dev).current_cells(cell_start, order);
  });
}

tlsph_status tlsph_dev_set_sweep_tiling(tlsph_dev* dev, tlsph_dev_sweep_tiling mode) {
  return guarded([&] {
    if (mode != TLSPH_SWEEP_TILING_AUTO && mode != TLSPH_SWEEP_TILING_STAGED && mode != TLSPH_SWEEP_TILING_STREAMED)
      throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "unknown sweep tiling");
    sys(dev).sweep_tiling = mode;
  });
}

tlsph_status tlsph_dev_set_sweep_blocking(tlsph_dev* dev, int columns, int phases) {
  return guarded([&] {
    if (columns < -1) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "sweep blocking: columns must be >= -1");
    sys(dev).sweep_block_w = columns;
    sys(dev).sweep_block_k = phases;
  });
}

tlsph_status tlsph_dev_grid_info(const tlsph_dev* dev, int* dims, double* origin, double* cell_size,
                                 int64_t* n_cells) {
  return guarded([&] {
    const DevSystem& s = sys(dev);
    for (int d = 0; d < s.D; ++d) {
      if (dims) dims[d] = s.dims[d];
      if (origin) origin[d] = s.origin[d];
    }
    if (cell_size) *cell_size = s.cutoff;
    if (n_cells) *n_cells = s.ncells;
  });
}

tlsph_status tlsph_dev_grid_cells(const tlsph_dev* dev, int32_t* cell_of, int64_t* cell_start,
                                  int32_t* cell_particles) {
  return guarded([&] { sys(dev).grid_cells(cell_of, cell_start, cell_particles); });
}

tlsph_status tlsph_dev_get_neighborhood(const tlsph_dev* dev, int64_t* offsets, int32_t* neighbor, double* r0_len,
                                        double* e0, double* dwdr0, double* pair_factor) {
  return guarded([&] { sys(dev).get_neighborhood(offsets, neighbor, r0_len, e0, dwdr0, pair_factor); });
}

tlsph_status tlsph_dev_correction_matrices(tlsph_dev* dev) {
  return guarded([&] { sys(dev).correction_matrices(); });
}

tlsph_status tlsph_dev_deformation_rate(tlsph_dev* dev) {
  return guarded([&] { sys(dev).deformation_rate(); });
}

tlsph_status tlsph_dev_update_density(tlsph_dev* dev) {
  return guarded([&] { sys(dev).update_density(); });
}

tlsph_status tlsph_dev_momentum_rhs(tlsph_dev* dev, const tlsph_dev_material* mat) {
  return guarded([&] {
    require_material(mat);
    sys(dev).momentum_rhs(tlsph_cuda::to_dmat(*mat));
  });
}

tlsph_status tlsph_dev_verlet_step(tlsph_dev* dev, const tlsph_dev_material* mat, double dt) {
  return guarded([&] {
    require_material(mat);
    sys(dev).verlet_step(tlsph_cuda::to_dmat(*mat), dt);
  });
}

tlsph_status tlsph_dev_apply_constraints(tlsph_dev* dev) {
  return guarded([&] { sys(dev).apply_constraints(); });
}

tlsph_status tlsph_dev_stable_dt(tlsph_dev* dev, const tlsph_dev_material* mat, double h, double* dt_acoustic) {
  return guarded([&] {
    require_material(mat);
    if (!dt_acoustic) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "output must not be null");
    *dt_acoustic = sys(dev).stable_dt(tlsph_cuda::to_dmat(*mat), h);
  });
}

tlsph_status tlsph_dev_kinetic_energy(tlsph_dev* dev, double* out) {
  return guarded([&] {
    if (!out) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "output must not be null");
    *out = sys(dev).kinetic_energy();
  });
}

tlsph_status tlsph_dev_check_finite(tlsph_dev* dev, uint64_t step) {
  return guarded([&] { sys(dev).check_finite(step); });
}

tlsph_status tlsph_dev_verlet_pass(tlsph_dev* dev, const tlsph_dev_material* mat, double dt, int pass) {
  return guarded([&] {
    require_material(mat);
    sys(dev).verlet_pass(tlsph_cuda::to_dmat(*mat), dt, pass);
  });
}

tlsph_status tlsph_dev_reduce_state(tlsph_dev* dev, int want_ke, int64_t check_step, double* out) {
  return guarded([&] {
    if (!out) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "out must not be null");
    sys(dev).reduce_owned(want_ke != 0, check_step, out);
  });
}

tlsph_status tlsph_dev_damping_sweep(tlsph_dev* dev, tlsph_dev_scheme scheme, double eta_tilde, double dt) {
  return guarded([&] { sys(dev).damping_sweep(scheme, eta_tilde, dt, 1); });
}

tlsph_status tlsph_dev_damping_sweeps(tlsph_dev* dev, tlsph_dev_scheme scheme, double eta_tilde, double dt,
                                      int count) {
  return guarded([&] {
    if (count < 0) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "count must be non-negative");
    sys(dev).damping_sweep(scheme, eta_tilde, dt, count);
  });
}

tlsph_status tlsph_dev_particle_split_update(tlsph_dev* dev, size_t i, double eta, double dt_half) {
  return guarded([&] { sys(dev).particle_split_update(static_cast<long long>(i), eta, dt_half); });
}

tlsph_status tlsph_dev_pairwise_split_update(tlsph_dev* dev, size_t i, int64_t slot, double eta, double dt_half) {
  return guarded([&] { sys(dev).pairwise_split_update(static_cast<long long>(i), slot, eta, dt_half); });
}

tlsph_status tlsph_dev_explicit_damping_accel(tlsph_dev* dev, double eta, double* out) {
  return guarded([&] {
    if (!out) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "output must not be null");
    sys(dev).explicit_damping_accel(eta, out);
  });
}

tlsph_status tlsph_dev_run(tlsph_dev* dev, const tlsph_dev_loop_params* params, tlsph_dev_loop_result* result) {
  return guarded([&] {
    if (!params || !result) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "params and result must not be null");
    sys(dev).run(*params, *result);
  });
}

// RandomSource (damping.hpp:41-50): std::mt19937_64, u = (x >> 11) * 2^-53.
tlsph_status tlsph_random_uniforms(uint64_t seed, size_t n, double* out) {
  return guarded([&] {
    if (!out && n) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "output must not be null");
    std::mt19937_64 gen(seed);
    for (size_t k = 0; k < n; ++k) out[k] = static_cast<double>(gen() >> 11) * 0x1.0p-53;
  });
}

// random_choice_eta (damping.cpp:29-34) applied n times to one stream.
tlsph_status tlsph_random_choice(double eta, double alpha, uint64_t seed, size_t n, double* out) {
  return guarded([&] {
    if (!(alpha > 0.0 && alpha <= 1.0))
      throw DevError(TLSPH_ERR_INVALID_ARGUMENT,
                     "random-choice probability must lie in (0, 1], got " + std::to_string(alpha));
    if (!out && n) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "output must not be null");
    std::mt19937_64 gen(seed);
    for (size_t k = 0; k < n; ++k) {
      const double phi = static_cast<double>(gen() >> 11) * 0x1.0p-53;
      out[k] = phi < alpha ? eta / alpha : 0.0;
    }
  });
}

double tlsph_dev_last_elapsed(const tlsph_dev* dev) { return dev ? dev->sys.last_elapsed : -1.0; }
int64_t tlsph_dev_last_run_steps(const tlsph_dev* dev) { return dev ? dev->sys.last_run_steps : -1; }
double tlsph_dev_last_run_time(const tlsph_dev* dev) { return dev ? dev->sys.last_run_t : -1.0; }

tlsph_status tlsph_dev_selftest_division(int64_t n, uint64_t seed, uint64_t* mismatches) {
  return guarded([&] {
    if (!mismatches) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "output must not be null");
    CK(cudaSetDevice(g_default_device));
    *mismatches = tlsph_cuda::selftest_division(n, seed);
  });
}

}  // extern "C"
