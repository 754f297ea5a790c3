// Shared device-side definitions for the sm_100a TL-SPH relaxation path.
//
// Layout (DESIGN.md §Data layout): particles live in CELL-SORTED order
// (stable counting sort by x-fastest cell key, ascending reference id inside
// a cell), every per-particle field is a separate fp64 array (SoA), matrices
// are D*D arrays indexed r*D+c. The reference-configuration CSR is stored in
// the same sorted row order; each row keeps the reference's ascending
// reference-j slot order so ordered reductions reproduce the reference sums.
//
// All device arithmetic is compiled with -fmad=false: no silent FMA
// contraction, so every +,-,*,/ and sqrt rounds exactly as the reference's
// x86-64 (no -march, SSE2) build does. Explicit __fma_rn is used only where
// a correctly-rounded result is proven (none in round 1).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "tlsph/tlsph.h"

namespace tlsph_cuda {

// ---------------------------------------------------------------- errors
struct DevError : std::runtime_error {
  tlsph_status status;
  DevError(tlsph_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw DevError(TLSPH_ERR_INTERNAL, std::string("CUDA error in ") + what + " (" + file + ":" +
                                           std::to_string(line) + "): " + cudaGetErrorString(e));
}
#define CK(expr) ::tlsph_cuda::cuda_check((expr), #expr, __FILE__, __LINE__)
#define CK_LAUNCH(what) ::tlsph_cuda::cuda_check(cudaGetLastError(), what, __FILE__, __LINE__)

// Device error sites (first failing site in program order wins; lowest
// reference index within a site), mirroring the reference's throw points.
enum ErrSite : int {
  ERR_DENSITY_PRE = 0,   // update_density before the half-kick (integrator.cpp:126 -> :60-78)
  ERR_MOMENTUM = 1,      // compute_momentum_rhs det check (integrator.cpp:89-103)
  ERR_DENSITY_POST = 2,  // update_density after dF/dt (integrator.cpp:144)
  ERR_NAN = 3,           // check_finite (runner.cpp:233-247)
  ERR_DEGENERATE = 4,    // compute_correction_matrices (integrator.cpp:30-40)
  ERR_COINCIDENT = 5,    // build_reference_neighborhoods (neighbors.cpp:110-112)
  ERR_NONFINITE_R0 = 6,  // build_cell_grid (neighbors.cpp:34-35)
  ERR_SITES = 8
};

// Device-resident scalars of the time loop (runner.cpp:341-391 locals).
struct DScalars {
  double t;
  double dt;
  double end_time;
  double last_dt;
  unsigned long long vmax_bits;  // max |v| as ordered bits (non-negative doubles)
  unsigned long long amax_bits;
  unsigned int block_counter;    // last-block-done counter of the reduction kernel
  int halt;                      // 1: done or failed; every loop kernel returns early
  int done;
  int failed;
  long long steps;               // completed steps
  int pending;                   // a step was started whose accounting is not done yet
  long long err_step;
  unsigned long long err_key[ERR_SITES];  // per-site min key (reference index, or packed key)
  double ke;                     // kinetic energy accumulator
  double ke_peak;
  int ke_stop;
  double ke_ratio;
  int stopped_on_ke;
  double params[8];              // loop constants: h, c, viscous bound, fixed_dt, ...
  // probe output at marks (runner.cpp:381-390)
  double next_mark;
  double interval;
  long long probe;               // sorted index of the probe particle, < 0: none
  double* probe_buf;             // 4 doubles per sample
  long long probe_cap;
  long long probe_count;
  int pause_on_mark;
  int paused;
};

// Device pointers of the sorted SoA system (passed by value to kernels).
struct DFields {
  long long n;
  int dim;
  double* r0[3];
  double* r[3];
  double* v[3];
  double* a[3];
  double* body[3];
  double* F[9];
  double* dFdt[9];
  double* B0[9];
  // per particle, packed for the momentum gather: P(F) B0 row-major (D x D), V0, padding to 16 B
  double* pbv;
  double* v4;  // 3D bodies with the interleaved slot copy: (v, V0) records for pass C (k_pack_v4)
  double* V0;
  double* m;
  double* minvf;  // RN(1/m), negated for clamped particles (flag travels with the TMA-staged mass)
  double* qf;     // per slot: pair_factor * RN(1/m_j), 0 for clamped j (FAST sweep)
  double* pkf;    // per slot, per (eta, dt): the pairwise factor b / (m_i m_j - (m_i + m_j) b) (sweep.cu)
  // uniform masses (every m equal): RN(1/m), and per slot the stencil index with bit 15 set for
  // a clamped j (the streamed FAST sweep forms qf = pf * minv_uniform from them); null otherwise
  const uint16_t* nlocf;
  // bank-spread rows (uniform masses, TLSPH_SWEEP_SPREAD): nlocf and this copy of pf hold every row
  // regrouped for conflict-free half-warp gathers; ghdr[i] = the row's group starts (k_spread_rows)
  const double* pfsp;
  const unsigned long long* ghdr;
  // dense rows (large bodies, build_spread_rows): the bank-spread rows again, each padded to
  // dense_r = 32 K slots (group g at 16 g; padding: pair factor 0, the group's first stencil index),
  // so lane l of iteration u reads slot 32 u + l of row i at i * dense_r with no header decode and
  // no predicate; null when not built
  const uint16_t* nld;
  const double* pfd;
  int dense_r;
  double minv_uniform;
  double v0_uniform;  // every V0 equal: that value (the FAST dF/dt pass skips the V0_j gather); 0 otherwise
  // x-slab peers (slabs.py): per particle of a column shared with a neighbouring slab, the
  // particle's index in that slab's arrays (-1: not shared; >= 0: right peer; <= -2: left
  // peer at -2 - index); the peers' velocity arrays (device memory reachable from here)
  int* peer_idx;
  double* peer_v[2][3];
  int peer_x[2];  // the columns adjoining each peer (left: x0, right: x1 - 1), -1 if none
  double* pfsum;  // per particle: sum of its pair factors, and of their squares, in slot order
  double* pfsq;   //   (FAST fold constants without a pass over the slots)
  long long* cell_slot;  // offs[cell_start[c]]: first CSR slot of cell c (ncells+1)
  // per-sweep particle-split constants (sweep.cu, k_sweep_folds)
  double* fdiag;  // sum_j b_ij - m_i
  double* fden;   // diag^2 + sum_j b_ij^2
  double* fy;     // RN(1 / den)
  double* rho0;
  double* rho;
  uint8_t* flag;
  // x-slab ownership (slabs.py): 1 for particles of the slab's own cell columns, 0 for its halo
  // columns; null when the system is not a slab (every particle owned). The TL-SPH passes and
  // reductions skip halo particles, whose state arrives from the owning slab.
  const uint8_t* own;
  int* perm;  // sorted -> reference index
  int* rank;  // reference -> sorted index
  // reference-configuration CSR in sorted row order
  long long* offs;
  int* nbr;  // sorted index of j
  double* r0_len;
  double* e0[3];
  double* dwdr0;
  // the same slots with each row re-ordered by ascending (cell-sorted) neighbour index: the FAST
  // neighbour passes B and C gather from neighbours grouped by cell (fewer cache lines per warp
  // load than the reference's ascending-reference-id order, which the ORDERED kernels keep)
  // (snbr/sdw/se0: built for bodies below 65,536 particles only, which run the eight-lane FAST
  // kernels). Slot-order neighbour passes: the slot arrays interleaved by groups of 32 consecutive
  // particles (slot k of particle i at ogbase[i / 32] + 32 k + i % 32), so the one-thread-per-
  // particle loops load coalesced; built for every body of >= 65,536 particles (both modes run the
  // one-thread kernels there) and for ORDERED mode on smaller ones (build_ordered_rows)
  const int* onbr;
  const double* odw;
  const double* oe0[3];
  const long long* ogbase;
  const int* snbr;
  const double* sdw;
  const double* se0[3];
  double* pf;
  uint16_t* nloc;  // index of j inside the staged 3^D stencil of i's cell
  // cell grid
  long long* cell_start;
  int dims[3];
  double origin[3];
  double cell;
  int has_body;
  // optional penalty contact plane (forces.hpp:13-39)
  int contact;
  double cp_point[3];
  double cp_normal[3];
  double cp_k;
};

// x-slab ownership: halo particles of a slab are read, never advanced, by the TL-SPH passes
__device__ __forceinline__ bool is_owned(const DFields& f, long long i) { return !f.own || f.own[i]; }

constexpr int kWarp = 32;
// 3D slot-order neighbour passes: (dW/dr0, e0) of a slot as one 32-byte record of the interleaved
// copy (DFields::odw holds 4 doubles per slot, oe0 unused); 0: four separate arrays (A/B)
#ifndef TLSPH_TL_SLOTREC
#define TLSPH_TL_SLOTREC 1
#endif
// 3D slot-order pass C gathers (v_j, V0_j) as one 32-byte record packed right before the pass
// (tlsph.cu k_pack_v4); 0: three or four 64-bit gathers from the component arrays (A/B)
#ifndef TLSPH_TL_V4
#define TLSPH_TL_V4 1
#endif
// FAST particle-split chain on bank-spread slot rows (state.cu k_spread_rows, sweep_chain.cuh);
// 0: rows in slot order (A/B)
#ifndef TLSPH_SWEEP_SPREAD
#define TLSPH_SWEEP_SPREAD 1
#endif
constexpr uint16_t kNoLocal = 0xFFFF;

// ---------------------------------------------------------------- small helpers
__device__ __forceinline__ unsigned long long ordered_bits(double x) {  // x >= 0
  return static_cast<unsigned long long>(__double_as_longlong(x));
}
__device__ __forceinline__ double from_ordered_bits(unsigned long long b) {
  return __longlong_as_double(static_cast<long long>(b));
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

template <int G>
__device__ __forceinline__ double group_sum(double x) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Sum over groups of G consecutive lanes (G = 4 or 8) with the fp64 tensor-core MMA: mma.sync
// m8n8k4 with B = ones gives every lane the sum of its four-lane group (lane 4r+k supplies
// A[r][k]); one xor level completes G = 8. Whole warp, converged. FAST summation order.
#ifndef TLSPH_GROUP_MMA
#define TLSPH_GROUP_MMA 1
#endif
template <int G>
__device__ __forceinline__ double group_sum_mma(double x) {
  static_assert(G == 4 || G == 8, "G");
  double r, unused;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
               : "=d"(r), "=d"(unused)
               : "d"(x), "d"(1.0), "d"(0.0), "d"(0.0));
  if (G == 8) r += __shfl_xor_sync(0xffffffffu, r, 4);
  return r;
}

template <int G>
__device__ __forceinline__ double group_sum_fast(double x) {
  if constexpr (TLSPH_GROUP_MMA && (G == 4 || G == 8)) return group_sum_mma<G>(x);
  else return group_sum<G>(x);
}

// ---------------------------------------------------------------- cell grid
// CellGrid::coords_of_position (neighbors.cpp:14-22) and linear_index
// (neighbors.hpp:32-36, x fastest).
template <int D>
__device__ __forceinline__ void cell_coords(const double* p, const double* origin, double cell, const int* dims,
                                            int* c) {
#pragma unroll
  for (int d = 0; d < D; ++d) {
    int idx = static_cast<int>(floor((p[d] - origin[d]) / cell));
    c[d] = idx < 0 ? 0 : (idx > dims[d] - 1 ? dims[d] - 1 : idx);
  }
}

template <int D>
__device__ __forceinline__ long long cell_linear(const int* c, const int* dims) {
  long long idx = c[D - 1];
#pragma unroll
  for (int d = D - 2; d >= 0; --d) idx = idx * dims[d] + c[d];
  return idx;
}

// The staged stencil of a cell: 3^(D-1) x-rows (dz, dy), each spanning cells
// x-1..x+1 clamped to the grid, which are contiguous in cell-sorted particle
// order. Segment k = (dz+1)*3 + (dy+1) in 3D, (dy+1) in 2D.
// Shared-memory layout: each segment is staged as the 16-byte aligned
// superset of its fp64 range (so it can be moved by one TMA bulk copy);
// particle g of segment k sits at base[k] + (g - start[k]), where base[k]
// already includes the 0/1 element alignment offset. `total` is the padded
// tile length.
template <int D>
struct Stencil {
  static constexpr int kSegs = D == 2 ? 3 : 9;
  long long start[kSegs];
  int len[kSegs];
  int base[kSegs];
  int total;
};

template <int D>
__device__ __forceinline__ void stencil_segments(const long long* cell_start, const int* dims, const int* c,
                                                 Stencil<D>& st) {
  const int xlo = c[0] > 0 ? c[0] - 1 : 0;
  const int xhi = c[0] + 1 < dims[0] ? c[0] + 1 : dims[0] - 1;
  int running = 0;
#pragma unroll
  for (int k = 0; k < Stencil<D>::kSegs; ++k) {
    const int dy = (D == 2 ? k : k % 3) - 1;
    const int dz = D == 2 ? 0 : k / 3 - 1;
    const int y = c[1] + dy;
    const int z = D == 3 ? c[2] + dz : 0;
    bool ok = y >= 0 && y < dims[1];
    if (D == 3) ok = ok && z >= 0 && z < dims[2];
    long long s = 0, e = 0;
    if (ok) {
      const long long row = D == 3 ? (static_cast<long long>(z) * dims[1] + y) * dims[0] : static_cast<long long>(y) * dims[0];
      s = cell_start[row + xlo];
      e = cell_start[row + xhi + 1];
    }
    st.start[k] = s;
    st.len[k] = static_cast<int>(e - s);
    const int par = static_cast<int>(s & 1);
    st.base[k] = running + par;
    running += st.len[k] > 0 ? ((st.len[k] + par + 1) & ~1) : 0;
  }
  st.total = running;
}

// ---------------------------------------------------------------- small matrices
// Same operation order as oracle/tlsph_oracle.hpp (Eigen fixed-size paths).
template <int D>
struct M {
  double c[D][D];
};

__device__ __forceinline__ double det(const M<2>& m) { return m.c[0][0] * m.c[1][1] - m.c[1][0] * m.c[0][1]; }
__device__ __forceinline__ double det(const M<3>& m) {
  return m.c[0][0] * (m.c[1][1] * m.c[2][2] - m.c[1][2] * m.c[2][1]) -
         m.c[0][1] * (m.c[1][0] * m.c[2][2] - m.c[1][2] * m.c[2][0]) +
         m.c[0][2] * (m.c[1][0] * m.c[2][1] - m.c[1][1] * m.c[2][0]);
}

__device__ __forceinline__ M<2> inverse(const M<2>& m) {
  const double invdet = 1.0 / det(m);
  M<2> r;
  r.c[0][0] = m.c[1][1] * invdet;
  r.c[1][0] = -m.c[1][0] * invdet;
  r.c[0][1] = -m.c[0][1] * invdet;
  r.c[1][1] = m.c[0][0] * invdet;
  return r;
}

__device__ __forceinline__ double cof3(const M<3>& m, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return m.c[i1][j1] * m.c[i2][j2] - m.c[i1][j2] * m.c[i2][j1];
}

__device__ __forceinline__ M<3> inverse(const M<3>& m) {
  const double c00 = cof3(m, 0, 0), c10 = cof3(m, 1, 0), c20 = cof3(m, 2, 0);
  const double dt = (c00 * m.c[0][0] + c10 * m.c[1][0]) + c20 * m.c[2][0];
  const double invdet = 1.0 / dt;
  M<3> r;
#pragma unroll
  for (int row = 0; row < 3; ++row)
#pragma unroll
    for (int col = 0; col < 3; ++col) r.c[row][col] = cof3(m, col, row) * invdet;
  return r;
}

template <int D>
__device__ __forceinline__ M<D> matmul(const M<D>& a, const M<D>& b) {
  M<D> o;
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int k = 0; k < D; ++k) {
      double s = a.c[r][0] * b.c[0][k];
#pragma unroll
      for (int q = 1; q < D; ++q) s = s + a.c[r][q] * b.c[q][k];
      o.c[r][k] = s;
    }
  return o;
}

template <int D>
__device__ __forceinline__ M<D> transpose(const M<D>& a) {
  M<D> t;
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int k = 0; k < D; ++k) t.c[r][k] = a.c[k][r];
  return t;
}

// One-sided Jacobi singular values, same routine as the oracle's stand-in for
// Eigen::JacobiSVD (only the boolean condition test consumes it).
template <int D>
__device__ __forceinline__ void singular_values(const M<D>& a, double* sv) {
  double u[D][D];
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int k = 0; k < D; ++k) u[r][k] = a.c[r][k];
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
#pragma unroll
    for (int p = 0; p < D - 1; ++p)
#pragma unroll
      for (int q = p + 1; q < D; ++q) {
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
#pragma unroll
        for (int r = 0; r < D; ++r) {
          alpha = alpha + u[r][p] * u[r][p];
          beta = beta + u[r][q] * u[r][q];
          gamma = gamma + u[r][p] * u[r][q];
        }
        if (gamma == 0.0 || fabs(gamma) <= 1e-300 || fabs(gamma) <= 1e-17 * sqrt(alpha * beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t);
        const double sn = cs * t;
#pragma unroll
        for (int r = 0; r < D; ++r) {
          const double up = u[r][p], uq = u[r][q];
          u[r][p] = cs * up - sn * uq;
          u[r][q] = sn * up + cs * uq;
        }
      }
    if (!rotated) break;
  }
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < D; ++r) s = s + u[r][k] * u[r][k];
    sv[k] = sqrt(s);
  }
  // descending
#pragma unroll
  for (int x = 0; x < D; ++x)
#pragma unroll
    for (int y = 0; y < D - 1 - x; ++y)
      if (sv[y] < sv[y + 1]) {
        const double tmp = sv[y];
        sv[y] = sv[y + 1];
        sv[y + 1] = tmp;
      }
}

// Material constants as kernel arguments (material.hpp:16-27).
struct DMaterial {
  int model;  // 0 linear Kirchhoff, 1 neo-Hookean
  double lambda, mu, c;
};

// second_pk (material.cpp:32-44); caller guarantees det(F) > 0.
template <int D>
__device__ __forceinline__ M<D> second_pk(const M<D>& F, double J, const DMaterial& mat) {
  const M<D> C = matmul(transpose(F), F);
  M<D> S;
  if (mat.model == 0) {
    M<D> g;
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int k = 0; k < D; ++k) g.c[r][k] = 0.5 * (C.c[r][k] - (r == k ? 1.0 : 0.0));
    double tr = g.c[0][0];
#pragma unroll
    for (int d = 1; d < D; ++d) tr = tr + g.c[d][d];
    const double lt = mat.lambda * tr;
    const double twomu = 2.0 * mat.mu;
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int k = 0; k < D; ++k) S.c[r][k] = lt * (r == k ? 1.0 : 0.0) + twomu * g.c[r][k];
    return S;
  }
  const M<D> Ci = inverse(C);
  const double ll = mat.lambda * log(J);
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int k = 0; k < D; ++k) S.c[r][k] = mat.mu * ((r == k ? 1.0 : 0.0) - Ci.c[r][k]) + ll * Ci.c[r][k];
  return S;
}

// doubles per packed record of DFields::pbv
template <int D>
__host__ __device__ constexpr int pbv_stride() { return D == 3 ? 10 : 6; }

// Layout of DFields::pbv: component c of particle p. Chunk-major: a chunk of every particle is
// contiguous, so the momentum pass's gather of a chunk for the 32 neighbours a warp holds touches
// few 128-byte lines (neighbour indices come in runs); an 80-byte record per particle made every
// chunk load touch every record's line. 3D (TLSPH_PBV_WIDE): two 32-byte chunks (components 0-3,
// 4-7) and one 16-byte chunk (8, 9), gathered by two 256-bit loads and one 128-bit load instead of
// five 128-bit loads (fewer L1 tag lookups, the pass's bound). 2D: three 16-byte chunks.
#ifndef TLSPH_PBV_WIDE
#define TLSPH_PBV_WIDE 1
#endif
template <int D>
__host__ __device__ __forceinline__ long long pbv_at(long long n, long long p, int c) {
#ifdef TLSPH_PBV_AOS
  return p * pbv_stride<D>() + c;
#else
  if (D == 3 && TLSPH_PBV_WIDE) return c < 8 ? 4 * ((c >> 2) * n + p) + (c & 3) : 8 * n + 2 * p + (c - 8);
  return 2 * ((c >> 1) * n + p) + (c & 1);
#endif
}

// The packed 3D record of particle j (TLSPH_PBV_WIDE layout) into rec[0..9].
__device__ __forceinline__ void pbv_gather3(const double* __restrict__ pbv, long long n, long long j, double* rec) {
  const double* q0 = pbv + 4 * j;
  const double* q1 = pbv + 4 * (n + j);
  // TLSPH_TL_GATHER_HINT=1 (A/B): the gathered records kept in L1 with evict_last priority
#if defined(TLSPH_TL_GATHER_HINT) && TLSPH_TL_GATHER_HINT == 1
#define TLSPH_PBV_LD "ld.global.nc.L1::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];"
#else
#define TLSPH_PBV_LD "ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
#endif
  asm volatile(TLSPH_PBV_LD : "=d"(rec[0]), "=d"(rec[1]), "=d"(rec[2]), "=d"(rec[3]) : "l"(q0));
  asm volatile(TLSPH_PBV_LD : "=d"(rec[4]), "=d"(rec[5]), "=d"(rec[6]), "=d"(rec[7]) : "l"(q1));
#undef TLSPH_PBV_LD
  const double2 x = __ldg(reinterpret_cast<const double2*>(pbv + 8 * n + 2 * j));
  rec[8] = x.x;
  rec[9] = x.y;
}

template <int D>
__device__ __forceinline__ M<D> load_mat(double* const* arr, long long i) {
  M<D> m;
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int k = 0; k < D; ++k) m.c[r][k] = arr[r * D + k][i];
  return m;
}

template <int D>
__device__ __forceinline__ void store_mat(double* const* arr, long long i, const M<D>& m) {
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int k = 0; k < D; ++k) arr[r * D + k][i] = m.c[r][k];
}

// Error recording: lowest key wins. Only `failed` is latched here; `halt`
// is raised at the next serial point (the step-start reduction) so every
// block of the detecting kernel still records its candidates and the
// reported index is the reference's lowest one.
__device__ __forceinline__ void record_error(DScalars* sc, int site, unsigned long long key) {
  atomicMin(&sc->err_key[site], key);
  atomicOr(&sc->failed, 1);
  __threadfence();
}

}  // namespace tlsph_cuda
