// Host-side owner of one device-resident particle system (the object behind
// the opaque tlsph_dev handle of include/tlsph/tlsph_dev.h).
#pragma once

#include <atomic>
#include <vector>

#include "common.cuh"
#include "tlsph/tlsph_dev.h"

namespace tlsph_cuda {

// Simple owning device buffer.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  size_t cap = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  // (Re)sizes to `count` elements; keeps the allocation when it is big enough.
  void alloc(size_t count) {
    if (p && count <= cap) {
      n = count;
      return;
    }
    release();
    n = count;
    cap = count;
    // 16 elements of slack: the sweep's TMA stages 16-byte aligned supersets
    // of particle/slot ranges, which may read just past the last element.
    if (count) CK(cudaMalloc(&p, (count + 16) * sizeof(T)));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cap = 0;
  }
};

struct SweepPlan;  // damping.cu

// bytes moved by field transfers between host memory and the device (state.cu)
extern std::atomic<unsigned long long> g_h2d_bytes, g_d2h_bytes;

// A slab's export for cross-process linking: its velocity arrays and colour-phase events as
// CUDA IPC handles (tlsph_dev_ipc_export); plain bytes, exchanged by the host.
struct IpcExport {
  static constexpr unsigned kMagic = 0x74736c32u;  // "tsl2"
  unsigned magic;
  int dim, device, nphase;
  long long n;                  // particles of the slab (the stress record's layout depends on it)
  cudaIpcMemHandle_t vel[3];
  cudaIpcMemHandle_t pbv;       // packed P B0 / V0 records (pass A output, pass B input)
  cudaIpcEventHandle_t ev[54];  // colour phases
  cudaIpcEventHandle_t hev[3];  // halo pushes: TLSPH_DEV_COLUMN_VELOCITY, _STRESS; [2] the mark (tlsph_dev_mark_ipc)
};
// A neighbour opened from its export (mapped arrays, its phase and halo events)
struct IpcPeer {
  std::vector<void*> mem;
  std::vector<cudaEvent_t> ev;
  cudaEvent_t hev[3] = {nullptr, nullptr, nullptr};
  double* pbv = nullptr;
  long long n = 0;
  void close();
};

class DevSystem {
 public:
  int D = 3;
  int device = 0;
  long long n = 0;
  double h = 0.0;
  double cutoff = 0.0;
  cudaStream_t stream = nullptr;
  tlsph_dev_reduction reduction = TLSPH_REDUCTION_FAST;
  tlsph_dev_sweep_tiling sweep_tiling = TLSPH_SWEEP_TILING_AUTO;

  // grid
  int dims[3] = {1, 1, 1};
  double origin[3] = {0, 0, 0};
  long long ncells = 0;
  int max_cell = 0;     // max particles per cell
  int max_stencil = 0;  // max particles in a staged 3^D stencil
  long long max_cell_slots = 0;  // max CSR slots owned by one cell
  int max_row = 0;               // max slots of one particle
  bool stencil_ok = true;
  // x-slab decomposition: an explicit (global) grid instead of the bounding
  // box of the local particles, and the cell-x range whose cells are sweep tasks
  bool grid_given = false;
  double given_origin[3] = {0, 0, 0};
  int given_dims[3] = {1, 1, 1};
  int task_x0 = 0, task_x1 = -1;  // -1: dims[0]
  std::vector<long long> cell_start_h;  // host copy, for column packing
  // per colour: the non-empty task cells (x in the task range), fuller cells first, so a
  // phase's longest chains get the first SM slots; colour b's list starts at colour_start[b]
  // fused halo exchange with neighbouring slabs (tlsph_dev_link_peer)
  DBuf<int> peer_idx;
  DBuf<uint8_t> own;  // x-slab ownership mask (set_task_range); empty: all owned
  double* peer_v[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
  int peer_x[2] = {-1, -1};
  DBuf<int> colour_cells;
  std::vector<long long> colour_start;
  // the same task cells ordered by x column (fuller first within a column), for the temporally
  // blocked sweep (sweep.cu, enqueue_sweep_blocked): colour b's cells of column x are
  // xcol_cells[xcol_start[b * (dims[0] + 1) + x] .. xcol_start[b * (dims[0] + 1) + x + 1])
  DBuf<int> xcol_cells;
  std::vector<long long> xcol_start;
  int sweep_block_w = -1, sweep_block_k = 0;  // tlsph_dev_set_sweep_blocking (-1: automatic)
  std::vector<int> xcol_cells_h;
  // the dataflow sweep's task queue (cell, phase), per-column prefix counts, counters (sweep.cu)
  DBuf<int2> flow_queue;
  DBuf<int> flow_pref, flow_done;
  DBuf<unsigned long long> flow_head;
  int flow_w = 0, flow_k = 0;
  long long flow_ntask = 0;

  // fields (sorted order)
  DBuf<double> r0[3], r[3], v[3], a[3], body[3];
  DBuf<double> F[9], dFdt[9], B0[9];
  DBuf<double> pbv;   // packed P B0 + V0 per particle (common.cuh)
  DBuf<double> v4;    // (v, V0) records of the 3D slot-order pass C (tlsph.cu k_pack_v4)
  DBuf<double> V0, m, minvf, rho0, rho;
  DBuf<long long> cell_slot;
  // per-sweep particle-split constants and the (eta, dt) they were formed for
  DBuf<double> fold_diag, fold_den, fold_y;
  bool fold_valid = false;
  DBuf<double> pkf;  // pairwise factors per slot (k_pair_factors), valid for (pkf_eta, pkf_dt)
  bool pkf_valid = false;
  double pkf_eta = 0.0, pkf_dt = 0.0;
  double fold_eta = 0.0, fold_dt = 0.0;
  int fold_mode = -1;  // reduction mode the fold constants were formed in
  DBuf<uint8_t> flag;
  DBuf<int> perm, rank;
  DBuf<long long> cell_start;
  bool has_body = false;
  bool contact = false;
  double cp_point[3] = {0, 0, 0}, cp_normal[3] = {0, 0, 0}, cp_k = 0.0;
  // resumable loop state (pause_on_mark)
  bool loop_paused = false;
  std::vector<unsigned char> loop_flags;  // drawn random-choice outcomes, one per step
  uint64_t loop_consumed = 0;             // outcomes used by executed steps
  double loop_el = 0.0, loop_dm = 0.0, loop_tot = 0.0;
  DBuf<double> probe_dev;

  // CSR
  long long nslots = 0;
  DBuf<long long> offs;
  DBuf<int> nbr;
  DBuf<double> r0_len, e0[3], dwdr0, pf;
  DBuf<double> qf;  // pf * RN(1/m_j), 0 for clamped j: the FAST sweep's per-slot mass factor
  DBuf<double> pf_sum, pf_sq;  // per-particle sums of pf and pf^2 (static)
  DBuf<int> snbr;              // rows in neighbour-index order (k_sorted_rows): FAST passes B, C
  // per-step re-sort by current-position cell (set_resort / enqueue_resort, state.cu)
  bool resort = false;
  DBuf<int> rs_key, rs_perm, rs_count, rs_fill, rs_maxc;
  DBuf<long long> rs_start, rs_sums, rs_sums2;
  void set_resort(bool on);
  void enqueue_resort();
  void current_cells(int64_t* cell_start_h, int32_t* order_ref) const;
  DBuf<double> sdw, se0[3];
  DBuf<int> onbr;              // ORDERED passes: group-interleaved slot copy (build_ordered_rows)
  DBuf<double> odw, oe0[3];
  DBuf<long long> ogbase;
  void build_ordered_rows();
  DBuf<uint16_t> nloc;
  DBuf<uint16_t> nlocf;       // uniform masses: nloc | 0x8000 for clamped j (refresh_minvf)
  DBuf<double> pfsp;          // bank-spread rows: pf in the order of nlocf's regrouped rows
  DBuf<unsigned long long> ghdr;  // ... and each row's group starts (k_spread_rows)
  DBuf<uint16_t> nld;         // dense rows (k_dense_rows): n x dense_r stencil indices ...
  DBuf<double> pfd;           // ... and pair factors; large bodies only
  int dense_r = 0;            // 32 K, 0: not built
  bool uniform_mass = false;  // every particle has the same mass
  double minv_uniform = 0.0;  // RN(1/m) then
  double v0_uniform = 0.0;    // every V0 equal (> 0): that value; 0 otherwise (refresh_v0_uniform)
  void refresh_v0_uniform();

  // scratch
  DBuf<DScalars> scal;
  DBuf<double> tmp;        // AoS staging for host transfers
  DBuf<int> flag_buf;      // put_record change detection
  DBuf<long long> tmp_i64;
  DBuf<int> tmp_i32;
  DBuf<double> red;        // reduction partials
  double last_elapsed = 0.0;
  long long last_run_steps = 0;  // completed steps of the last tlsph_dev_run (also on failure)
  double last_run_t = 0.0;

  DevSystem() = default;
  ~DevSystem();

  DFields fields() const;

  // construction (state.cu)
  void init_common(int dim, size_t n_, const double* r0_h, const double* V0_h, const double* rho0_h,
                   const uint8_t* cons_h, double h_);
  void build_neighbourhoods();
  void load_csr(const int64_t* offsets, const int32_t* neighbor, const double* r0_len_h, const double* e0_h,
                const double* dwdr0_h, const double* pf_h);
  void compute_sweep_stats();
  void refresh_minvf();  // also refreshes qf once the CSR exists
  void build_spread_rows();  // nlocf, pfsp, ghdr: bank-spread rows of the FAST chain (uniform masses)

  // transfers (state.cu)
  void set_field(int field, const double* host);
  void get_field(int field, double* host) const;
  // the caller's own record storage (tlsph_dev_put / _take / _refresh): vectors D doubles,
  // matrices D*D doubles row-major (layout 0) or column-major (layout 1: tlsph::Mat, Eigen);
  // TLSPH_FIELD_CONSTRAINED as one byte per particle. only_if_changed: upload, compare with the
  // resident copy on the device and keep it when bitwise equal (*changed = 0).
  void put_record(int field, const void* host, int layout, bool only_if_changed, int* changed);
  void take_record(int field, void* host, int layout) const;
  void grid_cells(int32_t* cell_of, int64_t* cell_start_h, int32_t* cell_particles) const;
  void get_neighborhood(int64_t* offsets, int32_t* neighbor, double* r0_len_h, double* e0_h, double* dwdr0_h,
                        double* pf_h) const;

  // errors
  void reset_errors();
  void raise_if_failed(const char* context);  // throws DevError with the reference message

  void sync() const { CK(cudaStreamSynchronize(stream)); }

  // integrator (tlsph.cu)
  void correction_matrices();
  void deformation_rate();
  void update_density();
  void momentum_rhs(const DMaterial& mat);
  void verlet_step(const DMaterial& mat, double dt);
  void verlet_pass(const DMaterial& mat, double dt, int pass);
  void reduce_owned(bool want_ke, long long check_step, double out[3]);
  void apply_constraints();
  double stable_dt(const DMaterial& mat, double h_);
  double kinetic_energy();
  void check_finite(uint64_t step);

  // damping (damping.cu)
  void damping_sweep(int scheme, double eta_tilde, double dt, int count);
  void enqueue_sweep(int scheme, double eta_tilde, double dt_fixed, bool dt_from_scalars);
  // builds what enqueue_sweep allocates on first use (the dataflow schedule), before a graph capture
  void prepare_sweep_schedule(int scheme);
  // one colour phase (pass 0 forward / 1 reverse, index-th colour of the pass)
  void enqueue_sweep_phase(int scheme, double eta_tilde, double dt_fixed, int pass, int index);
  std::vector<cudaEvent_t> phase_events;  // tlsph_dev_sweep_linked: one per colour phase (this device)
  void build_colour_lists();  // host sync: at construction and when the task range changes
  void build_own_mask();      // own[] from the task range (x-slab ownership)
  void link_peer(int side, DevSystem& peer);  // sweep.cu
  void link_peer_arrays(int side, const long long* peer_cell_start, double* const* peer_vel);
  // cross-process linking (tlsph_dev_ipc_*), sweep.cu
  void ensure_phase_events(bool interprocess);
  void ipc_export(IpcExport* out);
  void link_peer_ipc(int side, const IpcExport& peer, const long long* peer_cell_start);
  void sweep_phase_ipc(int scheme, double eta_tilde, double dt, int q, int wait_q);
  IpcPeer ipc_peer[2];
  cudaEvent_t halo_events[3] = {nullptr, nullptr, nullptr};  // interprocess: halo pushes (velocity, stress), mark
  void push_halo_ipc(int field);
  void wait_halo_ipc(int field);
  void mark_ipc();
  void wait_mark_ipc();
  void wait_phase_ipc(int q);
  cudaEvent_t timer_ev[2] = {nullptr, nullptr};  // tlsph_dev_timer_start / _stop
  bool phase_events_ipc = false;
  // x-slab halo columns (sweep.cu)
  long long column_count(int x) const;
  int column_width(int field) const;  // doubles per particle of a column field
  void pack_column(int field, int x, double* dev_dst);
  void unpack_column(int field, int x, const double* dev_src);
  void particle_split_update(long long i, double eta, double dt_half);
  void pairwise_split_update(long long i, long long slot, double eta, double dt_half);
  void explicit_damping_accel(double eta, double* out_host);

  // loop (loop.cu)
  void run(const tlsph_dev_loop_params& p, tlsph_dev_loop_result& res);

 private:
  void alloc_fields();
};

DMaterial to_dmat(const tlsph_dev_material& m);
unsigned long long selftest_division(long long n, unsigned long long seed);  // sweep.cu

// kernels shared across translation units
void launch_reduce_state(const DevSystem& s, bool with_finite, bool with_ke, bool dt_mode);
void sweep_linked(const std::vector<DevSystem*>& slabs, int scheme, double eta_tilde, double dt, int count);

}  // namespace tlsph_cuda

struct tlsph_dev {
  tlsph_cuda::DevSystem sys;
};
