/* Thin host <-> CUDA C ABI of the B200 hot path (libtlsph_cuda.so).
 *
 * This is the layer the C++ host code (and the Python mirror used by the
 * tests and bench.py) calls to reach the sm_100a kernels. It owns a
 * device-resident particle system in cell-sorted structure-of-arrays fp64
 * layout; every entry point takes and returns host data in REFERENCE
 * particle order (the order ParticleSystem<D> stores), so callers never see
 * the device permutation.
 *
 * Each function returns a tlsph_status (tlsph.h) and never throws; on
 * failure tlsph_dev_last_error() holds a message. Device-detected solver
 * failures carry the reference's status and message text:
 *   inverted element  -> TLSPH_ERR_INVERTED_ELEMENT   (integrator.cpp:66-77,91-103)
 *   NaN in v or r     -> TLSPH_ERR_NUMERICAL_FAILURE  (runner.cpp:233-247)
 *   degenerate B0 /
 *   coincident pair   -> TLSPH_ERR_DEGENERATE_GEOMETRY (integrator.cpp:30-40, neighbors.cpp:110-112)
 * CUDA runtime failures map to TLSPH_ERR_INTERNAL.
 *
 * Vectors are n*D doubles, matrices n*D*D doubles (row-major per particle).
 */
#ifndef TLSPH_DEV_H
#define TLSPH_DEV_H

#include <stddef.h>
#include <stdint.h>

#include "tlsph/tlsph.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tlsph_dev tlsph_dev;

/* Field selectors for tlsph_dev_set_field / tlsph_dev_get_field
 * (ParticleSystem<D> members, particle_system.hpp:15-59, plus the body term
 * of ExternalAccel<D>, forces.hpp:34-38). */
typedef enum tlsph_dev_field {
  TLSPH_FIELD_R0 = 0,
  TLSPH_FIELD_R = 1,
  TLSPH_FIELD_V = 2,
  TLSPH_FIELD_A = 3,
  TLSPH_FIELD_F = 4,
  TLSPH_FIELD_DFDT = 5,
  TLSPH_FIELD_B0 = 6,
  TLSPH_FIELD_V0 = 7,
  TLSPH_FIELD_M = 8,
  TLSPH_FIELD_RHO0 = 9,
  TLSPH_FIELD_RHO = 10,
  TLSPH_FIELD_BODY = 11,
  TLSPH_FIELD_CONSTRAINED = 12 /* doubles 0/1 on the wire */
} tlsph_dev_field;

/* DampingScheme (damping.hpp:12) */
typedef enum tlsph_dev_scheme {
  TLSPH_SCHEME_EXPLICIT = 0,
  TLSPH_SCHEME_PARTICLE_SPLIT = 1,
  TLSPH_SCHEME_PAIRWISE_SPLIT = 2
} tlsph_dev_scheme;

/* Reduction order of neighbour sums.
 * ORDERED: every per-particle sum is a left fold over the CSR slots in
 *          ascending reference-j order, exactly as the reference loops, so
 *          damping/neighbour/B0/dF/dt results are bit-identical to the CPU
 *          reference arithmetic. Used by the parity tests.
 * FAST:    lanes split the slots and combine with warp shuffles (<= 1e-15
 *          relative per sum; the 1e-10 north_star class). Default. */
typedef enum tlsph_dev_reduction { TLSPH_REDUCTION_FAST = 0, TLSPH_REDUCTION_ORDERED = 1 } tlsph_dev_reduction;

/* Material (material.hpp:16-27): model 0 = linear Kirchhoff, 1 = neo-Hookean. */
typedef struct tlsph_dev_material {
  int model;
  double lambda, mu, K, G, E, nu, rho0, c;
} tlsph_dev_material;

const char* tlsph_dev_last_error(void);

/* Number of visible CUDA devices (0 without a GPU); never fails. */
int tlsph_dev_device_count(void);

/* Selects the CUDA device that subsequently created handles live on (one
 * process per GPU: pass LOCAL_RANK). Each handle remembers its device and
 * re-selects it on every call. Default 0. */
tlsph_status tlsph_dev_select_device(int ordinal);

/* Creates a device system from reference-order host arrays and runs the GPU
 * splitting cell-linked-list build: bounding box, cell keys, stable counting
 * sort into cells (build_cell_grid, neighbors.cpp:24-59), implicit 3^D
 * colouring (block_decompose, :61-77) and the reference-configuration CSR
 * with cached pair quantities (build_reference_neighborhoods, :79-141) for
 * cutoff = 2h. constrained may be NULL. B0 is left at identity. */
tlsph_status tlsph_dev_create(int dim, size_t n, const double* r0, const double* V0, const double* rho0,
                              const uint8_t* constrained, double h, tlsph_dev** out);

/* Same, but with a caller-built CSR (reference order) instead of the GPU
 * neighbour build; for hand-built rigs. The cell grid is still built from r0
 * with cutoff 2h so sweeps work when the CSR respects the 3^D stencil. */
tlsph_status tlsph_dev_create_with_csr(int dim, size_t n, const double* r0, const double* V0, const double* rho0,
                                       const uint8_t* constrained, double h, const int64_t* offsets,
                                       const int32_t* neighbor, const double* r0_len, const double* e0,
                                       const double* dwdr0, const double* pair_factor, tlsph_dev** out);

/* Cell grid only (build_cell_grid, neighbors.cpp:24-59): bins `positions`
 * with cell = cutoff; no neighbourhood is built, so coincident points are
 * allowed. Query it with tlsph_dev_grid_info / tlsph_dev_grid_cells. */
tlsph_status tlsph_dev_create_grid(int dim, size_t n, const double* positions, double cutoff, tlsph_dev** out);

/* One x-slab of a decomposed body: the local particles
 * (owned cell columns plus one halo column each side, ascending reference id)
 * binned in the GLOBAL cell grid (origin, dims; cell = 2h) so cell indices,
 * colours and in-cell order are those of the undivided body; neighbourhoods
 * are built on the GPU from the local particles. */
tlsph_status tlsph_dev_create_in_grid(int dim, size_t n, const double* r0, const double* V0, const double* rho0,
                                      const uint8_t* constrained, double h, const double* origin, const int* dims,
                                      tlsph_dev** out);
/* The slab's own cell columns [x0, x1) (default: the whole grid): they are its
 * sweep tasks, and the TL-SPH passes and reductions advance only the particles
 * of these columns (the halo columns' state arrives from their owners). */
tlsph_status tlsph_dev_set_task_range(tlsph_dev* dev, int x0, int x1);
/* One colour phase of strang_damping_sweep (damping.cpp:125-182): pass 0 is
 * the forward leg (colour `index` ascending), pass 1 the reverse leg; the
 * 2 * 3^D phases in order equal tlsph_dev_damping_sweep. Synchronous. */
tlsph_status tlsph_dev_damping_phase(tlsph_dev* dev, tlsph_dev_scheme scheme, double eta_tilde, double dt, int pass,
                                     int index);
/* Halo exchange of a slab system: velocities of the particles of cell column
 * x, component-major (D x count doubles), in (z, y, in-cell) order, which is
 * the same on every slab that holds the column. Device buffers; synchronous.
 * tlsph_dev_column_count returns -1 on error. */
/* Fused exchange: after this call the sweep phases of `dev` also store the new
 * velocities of the columns it shares with `peer` (side 0: the slab to its
 * left, 1: to its right) directly into `peer`'s arrays (peer access over
 * NVLink when the slabs live on different GPUs), so no pack/unpack is needed;
 * the caller only orders the phases of all slabs (a barrier per phase). */
tlsph_status tlsph_dev_link_peer(tlsph_dev* dev, int side, tlsph_dev* peer);
/* `count` sweeps over peer-linked slabs held by this process (slabs[r]'s
 * right neighbour is slabs[r+1]), enqueued at once with no host
 * synchronisation between phases: each slab's phases run on its own stream
 * (its GPU), and before phase q+1 a slab's stream waits on the phase-q events
 * of its two neighbours -- the per-phase barrier of the fused exchange, kept on
 * the devices. Returns after the last phase; tlsph_dev_last_elapsed(slabs[0])
 * then holds the device time of the whole call. Results equal the sweeps of
 * the undivided body bit for bit (ORDERED and FAST). */
/* Cross-process linking (one process per GPU, e.g. under torchrun). A slab
 * exports its velocity arrays and colour-phase events as CUDA IPC handles in an
 * opaque blob of tlsph_dev_ipc_size() bytes; the host hands the blobs and the
 * cell tables (tlsph_dev_grid_cells' cell_start, ncells + 1 entries) to the
 * neighbours, which open and link them (the fused exchange of
 * tlsph_dev_link_peer, across processes). tlsph_dev_sweep_phase_ipc then
 * enqueues colour phase q (0 .. 2*3^D - 1: forward leg, then the reverse leg)
 * asynchronously: the slab's stream first waits on the linked neighbours'
 * events of phase wait_q (-1: none), runs the phase and records its own phase-q
 * event. The caller must only request a wait on a phase its neighbours have
 * already enqueued (a host-side counter per slab suffices; see slabs.py).
 * tlsph_dev_synchronize waits for the slab's stream. */
size_t tlsph_dev_ipc_size(void);
tlsph_status tlsph_dev_ipc_export(tlsph_dev* dev, void* blob);
tlsph_status tlsph_dev_link_peer_ipc(tlsph_dev* dev, int side, const void* peer_blob, const int64_t* peer_cell_start);
tlsph_status tlsph_dev_sweep_phase_ipc(tlsph_dev* dev, tlsph_dev_scheme scheme, double eta_tilde, double dt, int q,
                                       int wait_q);
tlsph_status tlsph_dev_synchronize(tlsph_dev* dev);
/* Device time of a span of work on the slab's stream: tlsph_dev_timer_start
 * records a start event, tlsph_dev_timer_stop records the end, waits for it and
 * returns the elapsed seconds (negative on error). */
tlsph_status tlsph_dev_timer_start(tlsph_dev* dev);
double tlsph_dev_timer_stop(tlsph_dev* dev);
tlsph_status tlsph_dev_sweep_linked(tlsph_dev* const* slabs, int nslabs, tlsph_dev_scheme scheme, double eta_tilde,
                                    double dt, int count);
int64_t tlsph_dev_column_count(const tlsph_dev* dev, int x);
tlsph_status tlsph_dev_pack_column(tlsph_dev* dev, int x, double* device_dst);
tlsph_status tlsph_dev_unpack_column(tlsph_dev* dev, int x, const double* device_src);
/* The same for a named column field, component-major (width x count doubles):
 * VELOCITY (width D; the sweep's and pass C's halo), STRESS (width D*D + 1:
 * P B0 row-major and V0, the record pass B gathers, written by pass A). */
typedef enum tlsph_dev_column_field { TLSPH_DEV_COLUMN_VELOCITY = 0, TLSPH_DEV_COLUMN_STRESS = 1 } tlsph_dev_column_field;
int tlsph_dev_column_width(const tlsph_dev* dev, tlsph_dev_column_field field); /* -1 on error */
tlsph_status tlsph_dev_pack_column_field(tlsph_dev* dev, tlsph_dev_column_field field, int x, double* device_dst);
tlsph_status tlsph_dev_unpack_column_field(tlsph_dev* dev, tlsph_dev_column_field field, int x,
                                           const double* device_src);
/* Halo refresh of the full loop across processes (the exchange after verlet
 * passes A and B, with the same host ordering rule as the phases): push stores
 * this slab's owned boundary columns of `field` straight into the linked
 * neighbours' halo copies and records the slab's halo event; wait makes the
 * slab's stream wait on the neighbours' halo events of `field` (their pushes
 * into this slab). Both asynchronous. */
tlsph_status tlsph_dev_push_halo_ipc(tlsph_dev* dev, tlsph_dev_column_field field);
tlsph_status tlsph_dev_wait_halo_ipc(tlsph_dev* dev, tlsph_dev_column_field field);
/* Data-free ordering points of the cross-process protocol (same host counter
 * rule as the halo pushes). mark records this slab's mark event after all work
 * enqueued so far; wait_mark makes the slab's stream wait on the neighbours'
 * marks. A sweep starts with mark + wait_mark, so its first phase cannot store
 * into a neighbour that is still reading its velocities (verlet pass C).
 * wait_phase(q) makes the stream wait on the neighbours' phase-q events: a
 * sweep ends with wait_phase(last), so no neighbour store into this slab is
 * still in flight when the caller reads it. All asynchronous. */
tlsph_status tlsph_dev_mark_ipc(tlsph_dev* dev);
tlsph_status tlsph_dev_wait_mark_ipc(tlsph_dev* dev);
tlsph_status tlsph_dev_wait_phase_ipc(tlsph_dev* dev, int q);

void tlsph_dev_destroy(tlsph_dev* dev);

size_t tlsph_dev_size(const tlsph_dev* dev);
int tlsph_dev_dim(const tlsph_dev* dev);
int64_t tlsph_dev_slot_count(const tlsph_dev* dev);

tlsph_status tlsph_dev_set_field(tlsph_dev* dev, tlsph_dev_field field, const double* host);
tlsph_status tlsph_dev_get_field(const tlsph_dev* dev, tlsph_dev_field field, double* host);
tlsph_status tlsph_dev_set_reduction(tlsph_dev* dev, tlsph_dev_reduction mode);
/* Transfers in the caller's own per-particle record storage (reference
 * order), the form the C++ operator API moves ParticleSystem<D> fields in
 * without repacking: a vector field is D doubles per particle, a matrix field
 * D*D doubles, row-major (TLSPH_LAYOUT_ROW_MAJOR) or column-major
 * (TLSPH_LAYOUT_COL_MAJOR: tlsph::Mat<D>, Eigen's storage order);
 * TLSPH_FIELD_CONSTRAINED is one byte (0/1) per particle here.
 * tlsph_dev_refresh uploads, compares bitwise with the resident copy on the
 * device and keeps it when equal (*changed = 0), so derived per-particle data
 * (inverse masses, clamp bits, fold constants) is rebuilt only when the
 * caller really changed the field. For TLSPH_FIELD_R0 a difference is an
 * error (the cell order is built from r0). A null host array for
 * TLSPH_FIELD_BODY removes the body term (ExternalAccel<D>::body empty). */
typedef enum tlsph_dev_layout { TLSPH_LAYOUT_ROW_MAJOR = 0, TLSPH_LAYOUT_COL_MAJOR = 1 } tlsph_dev_layout;
tlsph_status tlsph_dev_put(tlsph_dev* dev, tlsph_dev_field field, const void* host, int layout);
tlsph_status tlsph_dev_refresh(tlsph_dev* dev, tlsph_dev_field field, const void* host, int layout, int* changed);
tlsph_status tlsph_dev_take(const tlsph_dev* dev, tlsph_dev_field field, void* host, int layout);
/* Cumulative bytes moved between host memory and the device by the field
 * transfers of all handles of this process (set/get_field, put/refresh/take). */
void tlsph_dev_transfer_bytes(uint64_t* h2d, uint64_t* d2h);
/* Page-locks (cudaHostRegister) a caller-owned host range so field transfers from and into it run
 * as direct DMA; idempotent per range. Unregister before the memory is freed. */
tlsph_status tlsph_dev_host_register(void* host, size_t bytes);
tlsph_status tlsph_dev_host_unregister(void* host);


/* Per-step re-sort (BASELINE cfg4): with `on`, every step of tlsph_dev_run
 * first rebuilds a storage permutation keyed by each particle's CURRENT-position
 * cell (the r0 grid, out-of-grid positions clamped to border cells): cell_start
 * and the particles of each cell in ascending storage order. The colouring,
 * neighbourhoods and sweep order stay r0-based, so no result changes; the
 * rebuild's time is part of the step. tlsph_dev_current_cells returns the last
 * one: cell_start (ncells + 1) and the reference ids in current-cell order (n). */
tlsph_status tlsph_dev_set_resort(tlsph_dev* dev, int on);
/* Completed steps and time of the last tlsph_dev_run, also when it stopped on an
 * error (inverted element, NaN): the step the reference would have reported. */
int64_t tlsph_dev_last_run_steps(const tlsph_dev* dev);
double tlsph_dev_last_run_time(const tlsph_dev* dev);
tlsph_status tlsph_dev_current_cells(const tlsph_dev* dev, int64_t* cell_start, int32_t* order);

/* Where the FAST particle-split sweep keeps a cell's slot block (pair factors,
 * stencil indices) while its chain runs: staged in shared memory (four to six
 * cells per SM; the form for colours of up to two waves of staged tiles, e.g.
 * 600-1,500 cells) or streamed from L2 (a tile of stencil velocities only,
 * 15 cells per SM; the throughput form for large bodies). AUTO picks by the
 * colour's cell count.
 * Results are identical in every mode. */
typedef enum tlsph_dev_sweep_tiling {
  TLSPH_SWEEP_TILING_AUTO = 0,
  TLSPH_SWEEP_TILING_STAGED = 1,
  TLSPH_SWEEP_TILING_STREAMED = 2
} tlsph_dev_sweep_tiling;
tlsph_status tlsph_dev_set_sweep_tiling(tlsph_dev* dev, tlsph_dev_sweep_tiling mode);

/* Temporal blocking of the colour-phase schedule over x-column chunks: phases are run k at a time,
 * each chunk of `columns` cell columns through an upright trapezoid (narrowing by 2 columns per
 * phase) and each chunk boundary through the inverted one, so a chunk's velocities stay in L2
 * across k phases. Every cell task sees the inputs of the phase-by-phase order: results are
 * bitwise identical. FAST particle split runs it as one persistent dataflow launch (per-column
 * completion counters), other schemes/modes as column-range launches. columns = -1: automatic
 * (the phase-by-phase order: blocking measured slower on this B200); columns = 0:
 * off; phases <= 0 with columns > 0: columns / 4. Ignored for x-slabs (task range or peers). */
tlsph_status tlsph_dev_set_sweep_blocking(tlsph_dev* dev, int columns, int phases);

/* Penalty contact plane of ExternalAccel<D> (forces.hpp:13-39): a_i +=
 * stiffness * max(0, -(r_i - point).normal) / m_i * normal, evaluated at the
 * current position inside the momentum RHS. stiffness <= 0 removes it. */
tlsph_status tlsph_dev_set_contact_plane(tlsph_dev* dev, const double* point, const double* normal,
                                         double stiffness);

/* CellGrid<D> (neighbors.hpp:18-48): dims[D], origin[D], cell_size, number of cells. */
tlsph_status tlsph_dev_grid_info(const tlsph_dev* dev, int* dims, double* origin, double* cell_size,
                                 int64_t* n_cells);
/* cell_of[n] (reference order); cell_start[n_cells+1]; cell_particles[n] =
 * reference ids of each cell in ascending order. */
tlsph_status tlsph_dev_grid_cells(const tlsph_dev* dev, int32_t* cell_of, int64_t* cell_start,
                                  int32_t* cell_particles);
/* ReferenceNeighborhood<D> (neighbors.hpp:67-82) in reference order. Any
 * output may be null; with every slot array null only the row offsets are
 * produced (no per-slot conversion). */
tlsph_status tlsph_dev_get_neighborhood(const tlsph_dev* dev, int64_t* offsets, int32_t* neighbor, double* r0_len,
                                        double* e0, double* dwdr0, double* pair_factor);

/* ---- operators (reference operator API, integrator.hpp / damping.hpp) ---- */
tlsph_status tlsph_dev_correction_matrices(tlsph_dev* dev);                 /* integrator.cpp:12-42 */
tlsph_status tlsph_dev_deformation_rate(tlsph_dev* dev);                    /* integrator.cpp:44-58 */
tlsph_status tlsph_dev_update_density(tlsph_dev* dev);                      /* integrator.cpp:60-78 */
tlsph_status tlsph_dev_momentum_rhs(tlsph_dev* dev, const tlsph_dev_material* mat); /* :80-116 */
tlsph_status tlsph_dev_verlet_step(tlsph_dev* dev, const tlsph_dev_material* mat, double dt); /* :118-152 */
tlsph_status tlsph_dev_apply_constraints(tlsph_dev* dev);                   /* particle_system.hpp:51-58 */
/* One pass of verlet_step (integrator.cpp:118-152) as the device loop fuses it:
 * 0 = A (density from J^n, half-kick of F and r, constraints, P B0 record),
 * 1 = B (momentum RHS + kick + constraints), 2 = C (dF/dt, density from
 * J^(n+1/2), half-kick, constraints). Passes 0, 1, 2 in order equal
 * tlsph_dev_verlet_step; an x-slab driver exchanges halo columns between them. */
tlsph_status tlsph_dev_verlet_pass(tlsph_dev* dev, const tlsph_dev_material* mat, double dt, int pass);
/* |v|max, |a|max (stable_dt's inputs, integrator.cpp:154-169) and, when
 * want_ke, the kinetic energy (:171-178) over the owned particles into out[3];
 * check_step >= 0 also runs check_finite (runner.cpp:233-247) for that step.
 * A slab driver combines them across slabs (max, max, sum). */
tlsph_status tlsph_dev_reduce_state(tlsph_dev* dev, int want_ke, int64_t check_step, double* out);
/* stable_dt (integrator.cpp:154-169): writes 0.6*min(h/(c+|v|max), sqrt(h/|a|max)). */
tlsph_status tlsph_dev_stable_dt(tlsph_dev* dev, const tlsph_dev_material* mat, double h, double* dt_acoustic);
tlsph_status tlsph_dev_kinetic_energy(tlsph_dev* dev, double* out);        /* integrator.cpp:171-178 */
/* check_finite (runner.cpp:233-247) with the reference message for `step`. */
tlsph_status tlsph_dev_check_finite(tlsph_dev* dev, uint64_t step);

/* strang_damping_sweep (damping.cpp:125-182): colour-scheduled forward +
 * mirrored reverse pass of the local implicit operator at dt/2. eta_tilde
 * == 0 returns immediately; the explicit scheme is rejected. */
tlsph_status tlsph_dev_damping_sweep(tlsph_dev* dev, tlsph_dev_scheme scheme, double eta_tilde, double dt);
/* `count` back-to-back sweeps with fixed eta_tilde and dt (the damping-only
 * benchmark); same result as calling the above count times. */
tlsph_status tlsph_dev_damping_sweeps(tlsph_dev* dev, tlsph_dev_scheme scheme, double eta_tilde, double dt,
                                      int count);
/* particle_split_update / pairwise_split_update on one particle (damping.cpp:53-106). */
tlsph_status tlsph_dev_particle_split_update(tlsph_dev* dev, size_t i, double eta, double dt_half);
tlsph_status tlsph_dev_pairwise_split_update(tlsph_dev* dev, size_t i, int64_t slot, double eta, double dt_half);
/* explicit_damping_accel (damping.cpp:36-51); out is n*D, reference order. */
tlsph_status tlsph_dev_explicit_damping_accel(tlsph_dev* dev, double eta, double* out);

/* ---- device-resident time loop (runner.cpp:341-391) ---- */
typedef struct tlsph_dev_loop_params {
  tlsph_dev_material material;
  double h;              /* smoothing length */
  double eta;            /* damping viscosity (0 disables damping) */
  double alpha;          /* random-choice probability */
  int scheme;            /* tlsph_dev_scheme */
  uint64_t seed;         /* RandomSource seed of the damping stream */
  double end_time;       /* <= 0: unbounded (stop on max_steps) */
  uint64_t max_steps;    /* hard cap (0: unbounded, needs end_time > 0) */
  double fixed_dt;       /* > 0: use this dt instead of stable_dt */
  int elastic;           /* 1: verlet_step every step; 0: damping-only loop */
  int ke_stop;           /* 1: stop at the first step with KE < ke_ratio * peak KE after the peak */
  double ke_ratio;
  /* probe output (runner.cpp:381-390): every step whose t reaches the next
   * output mark appends (t, r[probe] - r0[probe]) to `probe_out`
   * (capacity `probe_capacity` samples of 4 doubles: t, u0, u1, u2). */
  int64_t probe_index;   /* reference index; < 0 disables probe output */
  double output_interval;
  double* probe_out;
  size_t probe_capacity;
  int pause_on_mark;     /* 1: return after each recorded mark (snapshots "all"); resume with resume = 1 */
  int resume;            /* 1: continue the previous loop, paused at a mark or stopped at max_steps
                          * (same eta~ stream, t, step count; max_steps counts from the start) */
} tlsph_dev_loop_params;

typedef struct tlsph_dev_loop_result {
  uint64_t steps;
  uint64_t damped_steps;
  double t;
  double last_dt;
  double elastic_seconds; /* device time of step_begin (stable_dt, checks, re-sort) + the elastic kernels */
  double damping_seconds; /* device time of the damping kernels */
  double total_seconds;   /* device time of the whole loop */
  double peak_ke;
  double final_ke;
  int stopped_on_ke;
  size_t probe_samples;  /* samples written to probe_out (cumulative across resumes) */
  int paused;            /* 1: stopped at an output mark with pause_on_mark set */
  uint64_t kernel_launches; /* kernels this call launched (graph kernel nodes per step kind) */
} tlsph_dev_loop_result;

/* Runs the loop with all state resident on the device; the eta~ sequence is
 * drawn on the host from RandomSource(seed) (damping.hpp:41-50), one draw per
 * step after the elastic step, exactly as runner.cpp:358-360. The initial
 * state must already be prepared (B0, momentum RHS, deformation rate), as
 * runner.cpp:306-312 does before its loop. */
tlsph_status tlsph_dev_run(tlsph_dev* dev, const tlsph_dev_loop_params* params, tlsph_dev_loop_result* result);

/* ---- x-slab groups across processes (one process per GPU; csrc/cuda/group.cu) ----
 * A body decomposed along x over the GLOBAL cell grid: each process creates its slab with
 * tlsph_dev_create_in_grid (the particles of its columns [x0 - 1, x1 + 1), ascending reference id)
 * and tlsph_dev_set_task_range(x0, x1), prepares it (runner.cpp:306-312) and joins a group. The
 * group links every slab to its x neighbours through CUDA IPC (colour-phase and halo stores go
 * straight into the neighbour's arrays; the barriers are stream waits on IPC events) and combines
 * the step scalars through the caller's communicator, so the owned particles follow the
 * undivided body's device loop bit for bit. */
typedef enum tlsph_group_op { TLSPH_GROUP_MAX = 0, TLSPH_GROUP_SUM = 1 } tlsph_group_op;
/* The caller's collective transport (MPI, torch.distributed, ...). Every call is made by all
 * ranks in the same order; return 0 on success. allgather: `bytes` from each rank into `recv`
 * (size x bytes, rank order). allreduce_f64: in place over `count` doubles. */
typedef struct tlsph_group_comm {
  void* ctx;
  int rank;
  int size;
  int (*allgather)(void* ctx, const void* send, size_t bytes, void* recv);
  int (*allreduce_f64)(void* ctx, double* values, int count, int op);
} tlsph_group_comm;
typedef struct tlsph_dev_group tlsph_dev_group;
/* Collective: exchanges the IPC exports and cell tables, creates the shared enqueue counters and
 * links the neighbours. The slab must outlive the group. */
tlsph_status tlsph_dev_group_create(tlsph_dev* slab, const tlsph_group_comm* comm, tlsph_dev_group** out);
/* Collective: `count` strang_damping_sweeps (damping.cpp:125-182) of the whole body. */
tlsph_status tlsph_dev_group_sweep(tlsph_dev_group* group, tlsph_dev_scheme scheme, double eta_tilde, double dt,
                                   int count);
/* Collective: the loop of runner.cpp:341-391 for params->max_steps steps (fixed step count: no
 * end_time, KE stop, probe or resume). result: steps, damped_steps, t, last_dt and, in
 * total_seconds, this rank's device time of the loop (the caller takes the max over ranks). */
tlsph_status tlsph_dev_group_run(tlsph_dev_group* group, const tlsph_dev_loop_params* params,
                                 tlsph_dev_loop_result* result);
/* Collective (a final barrier); frees the group, not the slab. */
void tlsph_dev_group_destroy(tlsph_dev_group* group);
/* Message of the last failed tlsph_dev_group_* / tlsph_group_* call on this thread. */
const char* tlsph_group_last_error(void);
/* Host-only pieces (no device): the slab planner (column ranges balanced by particle count, each
 * at least min_width wide; ranges[2r], ranges[2r+1] = x0, x1 of rank r; -1 if impossible), the
 * per-step dt the group loop forms from the combined |v|max, |a|max (k_step_begin's formula),
 * and a check of a communicator's allgather / allreduce. */
int tlsph_group_plan(const int64_t* column_counts, int ncol, int world, int min_width, int* ranges);
double tlsph_group_step_dt(const tlsph_dev_loop_params* params, int dim, double vmax, double amax);
tlsph_status tlsph_group_comm_selftest(const tlsph_group_comm* comm);

/* Host RNG helpers (damping.hpp:41-50, damping.cpp:29-34). */
tlsph_status tlsph_random_uniforms(uint64_t seed, size_t n, double* out);
tlsph_status tlsph_random_choice(double eta, double alpha, uint64_t seed, size_t n, double* out);

/* Timing helpers for bench.py: device time (CUDA events on the handle's
 * stream) of `count` sweeps / steps already enqueued by the calls above is
 * returned through these (seconds). */
double tlsph_dev_last_elapsed(const tlsph_dev* dev);

/* Device self-test of the corrected quotient RN(x/d) = q0 + r*y used where the
 * divisor is known ahead of the Gauss-Seidel chain: counts mismatches against
 * IEEE division over n random operand pairs (expected 0). */
tlsph_status tlsph_dev_selftest_division(int64_t n, uint64_t seed, uint64_t* mismatches);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* TLSPH_DEV_H */
