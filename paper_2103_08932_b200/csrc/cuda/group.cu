// x-slab groups across processes, driven from C (tlsph_dev_group_*, include/tlsph/tlsph_dev.h).
//
// One process per GPU holds one slab of a body decomposed along x over the GLOBAL cell grid
// (paper_2103_08932_b200/slabs.py states the same protocol in Python): the slab's
// device system is binned in the global grid (tlsph_dev_create_in_grid) and sweeps the cells of
// its own columns [x0, x1) (tlsph_dev_set_task_range). The group links each slab to its x
// neighbours through CUDA IPC, so
//   * every colour phase's kernels store the columns a slab shares with a neighbour straight into
//     the neighbour's velocity arrays (NVLink peer stores between GPUs), and the phase barrier is a
//     stream wait on the neighbours' IPC phase events -- no host synchronisation between phases;
//   * the TL-SPH step's two halo refreshes (the (P B0, V0) records after pass A, velocities after
//     pass B's kick) are peer pushes ordered the same way;
//   * stable_dt's |v|max, |a|max are combined with an all-reduce (max is exact, so dt is bitwise
//     the undivided body's), and the random-choice stream is replicated on every rank.
// Owned particles then follow the undivided device loop bit for bit (runner.cpp:341-391).
//
// Host-side ordering. cudaStreamWaitEvent binds to an event's most recent record at call time, so
// before a slab enqueues phase g with a wait on its neighbours' phase g-1 events, their enqueue
// counters must show g. The counters live in a small file in /dev/shm shared by the group's
// processes (each writes only its own slot). Collective set-up (IPC handles, cell tables, the file
// name) and the per-step scalars travel through the caller's communicator (tlsph_group_comm:
// MPI, torch.distributed, ...), so the library has no transport dependency of its own.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "tlsph/tlsph_dev.h"

namespace {

struct GroupError : std::runtime_error {
  tlsph_status status;
  GroupError(tlsph_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

void ok(tlsph_status s) {
  if (s != TLSPH_OK) throw GroupError(s, tlsph_dev_last_error());
}

void comm_ok(int rc, const char* what) {
  if (rc != 0) throw GroupError(TLSPH_ERR_INTERNAL, std::string("group communicator failed in ") + what);
}

// Per-rank enqueue counters shared through a /dev/shm file: slot r of `phase` / `halo` is written
// only by rank r; readers spin (bounded) until their neighbours reach a value.
class SharedCounters {
 public:
  SharedCounters() = default;
  SharedCounters(const SharedCounters&) = delete;
  SharedCounters& operator=(const SharedCounters&) = delete;
  ~SharedCounters() { close(); }

  void open(const std::string& name, int world, bool create) {
    name_ = name;
    world_ = world;
    bytes_ = sizeof(std::int64_t) * 2 * static_cast<size_t>(world);
    const int fd = shm_open(name.c_str(), create ? (O_CREAT | O_RDWR | O_EXCL) : O_RDWR, 0600);
    if (fd < 0) throw GroupError(TLSPH_ERR_IO, "slab group: cannot open shared counters " + name);
    if (create && ftruncate(fd, static_cast<off_t>(bytes_)) != 0) {
      ::close(fd);
      throw GroupError(TLSPH_ERR_IO, "slab group: cannot size shared counters " + name);
    }
    void* p = mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    ::close(fd);
    if (p == MAP_FAILED) throw GroupError(TLSPH_ERR_IO, "slab group: cannot map shared counters " + name);
    base_ = static_cast<std::int64_t*>(p);
    owner_ = create;
    if (create) std::memset(base_, 0, bytes_);
  }
  void close() {
    if (base_) munmap(base_, bytes_);
    base_ = nullptr;
    if (owner_) shm_unlink(name_.c_str());
    owner_ = false;
  }
  void set(int table, int rank, std::int64_t v) { slot(table, rank).store(v, std::memory_order_release); }
  void wait(int table, const std::vector<int>& ranks, std::int64_t v) const {
    const auto t0 = std::chrono::steady_clock::now();
    for (int r : ranks) {
      for (unsigned spin = 0; slot(table, r).load(std::memory_order_acquire) < v; ++spin) {
        if ((spin & 1023) == 1023) {
          if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60))
            throw GroupError(TLSPH_ERR_INTERNAL, "slab group: neighbour " + std::to_string(r) +
                                                     " did not reach step " + std::to_string(v) + " within 60 s");
          std::this_thread::yield();
        }
      }
    }
  }

 private:
  std::atomic<std::int64_t>& slot(int table, int rank) const {
    static_assert(sizeof(std::atomic<std::int64_t>) == sizeof(std::int64_t), "lock-free shared counter");
    return *reinterpret_cast<std::atomic<std::int64_t>*>(base_ + table * world_ + rank);
  }
  std::string name_;
  int world_ = 0;
  size_t bytes_ = 0;
  std::int64_t* base_ = nullptr;
  bool owner_ = false;
};

constexpr int kPhaseTable = 0, kHaloTable = 1;

}  // namespace

struct tlsph_dev_group {
  tlsph_dev* slab = nullptr;
  tlsph_group_comm comm{};
  int dim = 3, nphase = 54;
  std::vector<int> neighbours;
  SharedCounters counters;
  std::int64_t enqueued = 0, pushed = 0;

  void barrier() {
    char in = 0;
    std::vector<char> out(static_cast<size_t>(comm.size));
    comm_ok(comm.allgather(comm.ctx, &in, 1, out.data()), "barrier");
  }

  // A data-free ordering point: this slab's stream waits on its neighbours' work enqueued so far
  // (shares the halo counter sequence: every rank issues the same sequence of pushes and marks).
  void mark() {
    ok(tlsph_dev_mark_ipc(slab));
    counters.set(kHaloTable, comm.rank, ++pushed);
    counters.wait(kHaloTable, neighbours, pushed);
    ok(tlsph_dev_wait_mark_ipc(slab));
  }

  void halo(tlsph_dev_column_field field) {
    ok(tlsph_dev_push_halo_ipc(slab, field));
    counters.set(kHaloTable, comm.rank, ++pushed);
    counters.wait(kHaloTable, neighbours, pushed);
    ok(tlsph_dev_wait_halo_ipc(slab, field));
  }

  // `count` sweeps enqueued phase by phase (slabs.py IpcSlabSweep.sweep): the first phase is
  // ordered after the neighbours' preceding work by the mark, each later one by their previous
  // phase; the call returns once this slab's last phase ran and every neighbour store into it
  // landed.
  void sweep(tlsph_dev_scheme scheme, double eta_tilde, double dt, int count) {
    if (eta_tilde == 0.0 || count <= 0) return;
    mark();
    for (int k = 0; k < count; ++k)
      for (int q = 0; q < nphase; ++q) {
        const bool first = k == 0 && q == 0;
        if (!first) counters.wait(kPhaseTable, neighbours, enqueued);
        ok(tlsph_dev_sweep_phase_ipc(slab, scheme, eta_tilde, dt, q, first ? -1 : (q + nphase - 1) % nphase));
        counters.set(kPhaseTable, comm.rank, ++enqueued);
      }
    counters.wait(kPhaseTable, neighbours, enqueued);
    ok(tlsph_dev_wait_phase_ipc(slab, nphase - 1));
    ok(tlsph_dev_synchronize(slab));
  }

  // |v|max and |a|max combined with max, the kinetic energy with sum (tlsph_dev_reduce_state).
  void reduce(int want_ke, std::int64_t check_step, double out[3]) {
    ok(tlsph_dev_reduce_state(slab, want_ke, check_step, out));
    double mx[2] = {out[0], out[1]};
    comm_ok(comm.allreduce_f64(comm.ctx, mx, 2, TLSPH_GROUP_MAX), "allreduce(max)");
    out[0] = mx[0];
    out[1] = mx[1];
    if (want_ke) comm_ok(comm.allreduce_f64(comm.ctx, out + 2, 1, TLSPH_GROUP_SUM), "allreduce(sum)");
  }
};

namespace {

thread_local std::string g_group_error;

template <typename Fn>
tlsph_status group_guard(Fn&& fn) {
  try {
    fn();
    return TLSPH_OK;
  } catch (const GroupError& e) {
    g_group_error = e.what();
    return e.status;
  } catch (const std::exception& e) {
    g_group_error = e.what();
    return TLSPH_ERR_INTERNAL;
  }
}

}  // namespace

extern "C" {

const char* tlsph_group_last_error(void) { return g_group_error.c_str(); }

double tlsph_group_step_dt(const tlsph_dev_loop_params* p, int dim, double vmax, double amax) {
  // k_step_begin's dt (loop.cu): stable_dt (integrator.cpp:154-169) capped by the viscous bound
  // of the scheme (damping.cpp:12-27, runner.cpp:343-351)
  if (p->fixed_dt > 0.0) return p->fixed_dt;
  const double h = p->h;
  double bound = h / (p->material.c + vmax);
  if (amax > 0.0) {
    const double b2 = std::sqrt(h / amax);
    bound = b2 < bound ? b2 : bound;
  }
  double dt = 0.6 * bound;
  if (p->eta > 0.0 && (p->scheme == TLSPH_SCHEME_PARTICLE_SPLIT || p->scheme == TLSPH_SCHEME_EXPLICIT)) {
    const double nu = p->eta / (p->alpha * p->material.rho0);
    const double vb = (p->scheme == TLSPH_SCHEME_EXPLICIT ? 0.5 : 50.0) * h * h / (nu * dim);
    dt = vb < dt ? vb : dt;
  }
  return dt;
}

int tlsph_group_plan(const int64_t* column_counts, int ncol, int world, int min_width, int* ranges) {
  // contiguous column ranges balanced by particle count, each at least min_width wide (slabs.plan)
  if (world < 1 || ncol < min_width * world || !column_counts || !ranges) return -1;
  std::vector<long double> cum(static_cast<size_t>(ncol) + 1, 0.0L);
  std::vector<std::int64_t> icum(static_cast<size_t>(ncol) + 1, 0);
  for (int x = 0; x < ncol; ++x) icum[static_cast<size_t>(x) + 1] = icum[static_cast<size_t>(x)] + column_counts[x];
  const double total = static_cast<double>(icum[static_cast<size_t>(ncol)]);
  int prev = 0;
  ranges[0] = 0;
  for (int r = 1; r < world; ++r) {
    const double target = total * r / world;
    int x = 0;  // first x with cum[x] >= target (searchsorted, side left)
    while (x <= ncol && static_cast<double>(icum[static_cast<size_t>(x)]) < target) ++x;
    x = std::max(x, prev + min_width);
    x = std::min(x, ncol - min_width * (world - r));
    ranges[2 * r - 1] = x;
    ranges[2 * r] = x;
    prev = x;
  }
  ranges[2 * world - 1] = ncol;
  return 0;
}

tlsph_status tlsph_dev_group_create(tlsph_dev* slab, const tlsph_group_comm* comm, tlsph_dev_group** out) {
  if (!out) return TLSPH_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  return group_guard([&] {
    if (!slab || !comm || !comm->allgather || !comm->allreduce_f64 || comm->size < 1 || comm->rank < 0 ||
        comm->rank >= comm->size)
      throw GroupError(TLSPH_ERR_INVALID_ARGUMENT, "slab group: invalid slab or communicator");
    auto g = std::make_unique<tlsph_dev_group>();
    g->slab = slab;
    g->comm = *comm;
    int dims[3];
    double origin[3], cell = 0.0;
    int64_t ncells = 0;
    ok(tlsph_dev_grid_info(slab, dims, origin, &cell, &ncells));
    g->dim = tlsph_dev_dim(slab);
    g->nphase = 2 * (g->dim == 2 ? 9 : 27);
    const int rank = comm->rank, world = comm->size;
    for (int r : {rank - 1, rank + 1})
      if (r >= 0 && r < world) g->neighbours.push_back(r);
    // IPC exports and cell tables of every slab
    const size_t blob = tlsph_dev_ipc_size();
    std::vector<unsigned char> mine(blob), blobs(blob * static_cast<size_t>(world));
    ok(tlsph_dev_ipc_export(slab, mine.data()));
    comm_ok(comm->allgather(comm->ctx, mine.data(), blob, blobs.data()), "allgather(ipc)");
    const size_t nst = static_cast<size_t>(ncells) + 1;
    std::vector<int64_t> cs(nst), cs_all(nst * static_cast<size_t>(world));
    ok(tlsph_dev_grid_cells(slab, nullptr, cs.data(), nullptr));
    comm_ok(comm->allgather(comm->ctx, cs.data(), nst * sizeof(int64_t), cs_all.data()), "allgather(cells)");
    // the counter file: rank 0 names and creates it, the others open it after a barrier
    char name[64] = {};
    if (rank == 0) {
      std::random_device rd;
      std::snprintf(name, sizeof name, "/tlsph_group_%d_%08x%08x", static_cast<int>(getpid()), rd(), rd());
    }
    std::vector<char> names(sizeof name * static_cast<size_t>(world));
    comm_ok(comm->allgather(comm->ctx, name, sizeof name, names.data()), "allgather(name)");
    std::memcpy(name, names.data(), sizeof name);
    if (rank == 0) g->counters.open(name, world, true);
    g->barrier();
    if (rank != 0) g->counters.open(name, world, false);
    g->barrier();
    if (rank > 0)
      ok(tlsph_dev_link_peer_ipc(slab, 0, blobs.data() + blob * (rank - 1), cs_all.data() + nst * (rank - 1)));
    if (rank + 1 < world)
      ok(tlsph_dev_link_peer_ipc(slab, 1, blobs.data() + blob * (rank + 1), cs_all.data() + nst * (rank + 1)));
    g->barrier();  // every slab linked before any phase runs
    *out = g.release();
  });
}

tlsph_status tlsph_dev_group_sweep(tlsph_dev_group* g, tlsph_dev_scheme scheme, double eta_tilde, double dt,
                                   int count) {
  return group_guard([&] {
    if (!g) throw GroupError(TLSPH_ERR_INVALID_ARGUMENT, "null group");
    if (scheme != TLSPH_SCHEME_PARTICLE_SPLIT && scheme != TLSPH_SCHEME_PAIRWISE_SPLIT)
      throw GroupError(TLSPH_ERR_INVALID_ARGUMENT, "slab groups sweep the split schemes only");
    g->sweep(scheme, eta_tilde, dt, count);
  });
}

tlsph_status tlsph_dev_group_run(tlsph_dev_group* g, const tlsph_dev_loop_params* p, tlsph_dev_loop_result* res) {
  return group_guard([&] {
    if (!g || !p || !res) throw GroupError(TLSPH_ERR_INVALID_ARGUMENT, "null group, params or result");
    if (p->max_steps == 0 || p->end_time > 0.0 || p->ke_stop || p->probe_index >= 0 || p->resume)
      throw GroupError(TLSPH_ERR_INVALID_ARGUMENT,
                       "slab group loops run a fixed step count (max_steps > 0; no end_time, KE stop, probe or resume)");
    const auto scheme = static_cast<tlsph_dev_scheme>(p->scheme);
    const bool damping = p->eta > 0.0;
    if (damping && scheme != TLSPH_SCHEME_PARTICLE_SPLIT && scheme != TLSPH_SCHEME_PAIRWISE_SPLIT)
      throw GroupError(TLSPH_ERR_INVALID_ARGUMENT, "slab groups sweep the split schemes only");
    if (damping && !(p->alpha > 0.0 && p->alpha <= 1.0))
      throw GroupError(TLSPH_ERR_INVALID_ARGUMENT, "random-choice probability must lie in (0, 1]");
    *res = tlsph_dev_loop_result{};
    // RandomSource(seed) (damping.hpp:41-50): one draw per step, replicated on every rank
    std::mt19937_64 rng(p->seed);
    const double eta_tilde = damping ? p->eta / p->alpha : 0.0;
    ok(tlsph_dev_timer_start(g->slab));
    double t = 0.0, dt = 0.0, red[3];
    for (uint64_t k = 0; k < p->max_steps; ++k) {
      g->reduce(0, k > 0 ? static_cast<int64_t>(k) : -1, red);  // check_finite of the previous step
      dt = tlsph_group_step_dt(p, g->dim, red[0], red[1]);
      if (p->elastic) {
        ok(tlsph_dev_verlet_pass(g->slab, &p->material, dt, 0));
        g->halo(TLSPH_DEV_COLUMN_STRESS);
        ok(tlsph_dev_verlet_pass(g->slab, &p->material, dt, 1));
        g->halo(TLSPH_DEV_COLUMN_VELOCITY);
        ok(tlsph_dev_verlet_pass(g->slab, &p->material, dt, 2));
      }
      if (damping) {
        const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;  // random_choice_eta
        if (u < p->alpha) {
          g->sweep(scheme, eta_tilde, dt, 1);
          ++res->damped_steps;
        }
      }
      t = t + dt;
    }
    g->reduce(0, static_cast<int64_t>(p->max_steps), red);
    res->total_seconds = tlsph_dev_timer_stop(g->slab);
    res->steps = p->max_steps;
    res->t = t;
    res->last_dt = dt;
    // this rank's kernels, a lower bound: per step the reduction and passes A-C (3D: + the (v, V0)
    // pack), per damped step the fold constants and the 2 x 3^D colour phases; halo pushes not counted
    const uint64_t per_elastic = p->elastic ? (g->dim == 3 ? 4u : 3u) : 0u;
    const uint64_t phases = g->dim == 3 ? 54u : 18u;
    res->kernel_launches = p->max_steps * (1u + per_elastic) + res->damped_steps * (1u + phases);
  });
}

void tlsph_dev_group_destroy(tlsph_dev_group* g) {
  if (!g) return;
  try {
    g->barrier();  // no rank unlinks the counters while another still waits on them
  } catch (...) {
  }
  delete g;
}

tlsph_status tlsph_group_comm_selftest(const tlsph_group_comm* comm) {
  return group_guard([&] {
    if (!comm || !comm->allgather || !comm->allreduce_f64) throw GroupError(TLSPH_ERR_INVALID_ARGUMENT, "null comm");
    const int world = comm->size;
    const int64_t mine[2] = {comm->rank, 1000 + 7 * comm->rank};
    std::vector<int64_t> all(2 * static_cast<size_t>(world));
    comm_ok(comm->allgather(comm->ctx, mine, sizeof mine, all.data()), "allgather");
    for (int r = 0; r < world; ++r)
      if (all[2 * r] != r || all[2 * r + 1] != 1000 + 7 * r)
        throw GroupError(TLSPH_ERR_INTERNAL, "allgather returned rank " + std::to_string(r) + "'s data out of order");
    double mx[2] = {static_cast<double>(comm->rank), -static_cast<double>(comm->rank)};
    comm_ok(comm->allreduce_f64(comm->ctx, mx, 2, TLSPH_GROUP_MAX), "allreduce(max)");
    double s = 1.0 + comm->rank;
    comm_ok(comm->allreduce_f64(comm->ctx, &s, 1, TLSPH_GROUP_SUM), "allreduce(sum)");
    if (mx[0] != world - 1 || mx[1] != 0.0 || s != world * (world + 1) / 2.0)
      throw GroupError(TLSPH_ERR_INTERNAL, "allreduce returned wrong values");
  });
}

}  // extern "C"
