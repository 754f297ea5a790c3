// Colour-scheduled, operator-split implicit viscous damping sweep (the hot kernel).
//
// Reference: proj/src/tlsph/damping.cpp:53-182 (particle_split_update,
// pairwise_split_update, strang_damping_sweep), neighbors.cpp:143-174
// (block_sweep), neighbors.cpp:61-77 (3^D residue colouring).
//
// Per sweep: k_sweep_folds forms, for every particle, sum b and sum b^2
// (b = eta G dt/2), diag = sum b - m_i, denom = diag^2 + sum b^2 and
// RN(1/denom) -- in slot order (ORDERED) or from static per-particle sums of G
// and G^2 (FAST). They do not depend on the velocities, so they are computed
// once, fully parallel, and reused by all 2 x 3^D colour phases (and by later
// sweeps with the same eta, dt and mode). A constrained particle gets a NaN
// diagonal (never updated as i, damping.cpp:151).
//
// Per colour phase, one launch over the colour's non-empty cells, fuller cells
// first (DevSystem::build_colour_lists). Colour b holds the cells whose
// coordinates are congruent to b's residues mod 3; their 3^D stencils are
// disjoint (neighbors.hpp:50-52), so every cell is an independent task:
//
// k_sweep_fast (FAST particle split, the bench path): one warp per cell,
// chained to the previous phase by programmatic dependent launch.
//   1. staging: the cell's slot block (pair factor G, per-slot mass factor
//      G/m_j, stencil-local index), row offsets and fold constants by bulk
//      copies (TMA) and the stencil rows' addresses -- all static, before
//      griddepcontrol.wait; then the stencil velocities by per-lane cp.async;
//   2. the chain (sweep_chain.cuh): the cell's particles in order (ascending
//      id forward, descending on the reverse leg, damping.cpp:112-121), all D
//      components per lane, one transposed shuffle tree per particle;
//   3. write-back of the stencil rows by bulk stores (disjoint stencils: no
//      races), plus, for a slab, the columns shared with its neighbours
//      straight into their arrays (writeback_peers).
//
// k_sweep_phase (ORDERED particle split): one 128-thread CTA per cell with the
// same staging; warp d runs the chain of component d (the update is separable
// per component once diag and denom are known): lanes form the residual terms,
// lane 0 folds them in slot order (bit-exact).
//
// k_sweep_pairwise (pairwise split, damping.cpp:91-106, palindrome :171-176):
// one warp per cell, PDL-chained like k_sweep_fast, with per-slot factors
// b/(m_i m_j - (m_i+m_j) b) formed once per (eta, dt) by k_pair_factors.
// ORDERED: lanes 0..D-1 run the D components' pair chains in lockstep
// (bit-exact). FAST: each leg of a particle's palindrome is a warp scan of
// affine maps of v_i, so all pairs of a row are solved at once.
//
// Division. B200 IEEE fp64 division costs ~425 cycles of dependent latency
// (tools/fp64_latency.cu), so no division sits on the chain:
//   ORDERED: x/d with d known ahead uses y = RN(1/d) and one Markstein
//            correction, q0 = RN(x y), r = fma(-d, q0, x) (exact),
//            q = RN(q0 + r y) = RN(x/d) (Markstein's theorem for a correctly
//            rounded reciprocal; checked bit-for-bit against IEEE division by
//            tlsph_dev_selftest_division and the ORDERED parity tests);
//   FAST:    x * y (<= 1 ulp), within the 1e-10 north_star class.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <tuple>
#include <type_traits>
#include <utility>
#include <vector>

#include "stencil_tile.cuh"
#include "sweep_chain.cuh"
#include "system.cuh"
#include "tma.cuh"

namespace tlsph_cuda {

namespace {

// k_sweep_phase: one CTA of D warps per cell (warp d: component d)

// Launch chained to the preceding kernel by programmatic dependent launch.
template <typename... KArgs, typename... Args>
void launch_pdl_phase(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                      Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kernel, args...));
}

struct Phase {
  const int* cells;  // this launch's task cells (linear index), fuller first; blockIdx -> cell
  long long ncol;    // cells in this launch
  long long ncol_colour;  // cells in the whole colour (the staged/streamed choice follows it)
  int forward;
  int S;           // padded stencil tile length, multiple of 8
  int SC;          // max slots per cell, multiple of 8
  int MC;          // max particles per cell, even
  int MR;          // per-warp scratch (max slots per particle): pairwise k, ORDERED residual terms
  int fast;        // FAST particle-split tile: 1 no masses, per-slot mass factors instead; 2 (streamed) stencil 1/m;
                   // 3 uniform masses, neither (slot clamp bit)
  double eta;
  double dt;       // used when dt_from_scalars == 0
  int dt_from_scalars;
};

template <int D>
__host__ __device__ constexpr int colour_count() { return D == 2 ? 9 : 27; }
// Shared-memory tile of one cell; every section is a multiple of 16 bytes.
template <int D>
struct Tile {
  uint64_t* bar;
  long long* seg_start;  // per stencil row: first particle
  int* seg_len;
  int* seg_base;         // tile position of the first particle
  double* sv[D];         // stencil velocities
  double* sm;            // stencil masses
  double* smf;           // stencil signed RN(1/m) (negative: clamped)
  long long* soff;       // aligned superset of offs[p0..p1]
  double* sdiag;         // aligned supersets of the fold constants of p0..p1-1
  double* sden;
  double* sy;
  double* spf;           // aligned superset of the cell's pair factors
  double* sqf;           // FAST: aligned superset of the cell's pair_factor / m_j (0: clamped j)
  double* skf;           // pairwise scratch, D x MR
  uint16_t* snl;         // aligned superset of stencil-local neighbour indices
};

__host__ __device__ inline int mco(int MC) { return (MC + 4) & ~1; }
constexpr int kHeader = 16 + 16 * 9;  // barrier + spare word + segment table

template <int D>
__host__ __device__ inline size_t tile_bytes(int S, int SC, int MC, int MR, int fast) {
  size_t b = kHeader;
  b += sizeof(double) * (static_cast<size_t>(fast == 1 || fast == 3 ? D : fast == 2 ? D + 1 : D + 2) * S);
  b += sizeof(long long) * static_cast<size_t>(mco(MC));
  b += sizeof(double) * static_cast<size_t>(3 * mco(MC));
  b += sizeof(double) * static_cast<size_t>(SC + 2) * (fast == 1 ? 2 : 1);
  b += sizeof(double) * static_cast<size_t>(D * MR);
  b += sizeof(uint16_t) * static_cast<size_t>(SC + 16);
  return (b + 15) & ~static_cast<size_t>(15);
}

// Tile layout: header | v[D][S] | (m[S] | 1/m[S]) | offs | diag | den | y | pf | (qf) | pairwise scratch | nloc
// (the bracketed sections: masses for ORDERED / pairwise, qf for FAST)
template <int D>
__device__ inline Tile<D> carve(unsigned char* base, const Phase& ph) {
  Tile<D> t;
  const int mc = mco(ph.MC);
  t.bar = reinterpret_cast<uint64_t*>(base);
  t.seg_start = reinterpret_cast<long long*>(base + 16);
  t.seg_len = reinterpret_cast<int*>(base + 16 + 8 * 9);
  t.seg_base = reinterpret_cast<int*>(base + 16 + 12 * 9);
  double* d = reinterpret_cast<double*>(base + kHeader);
#pragma unroll
  for (int k = 0; k < D; ++k) t.sv[k] = d + static_cast<size_t>(k) * ph.S;
  double* after_v = d + static_cast<size_t>(D) * ph.S;
  if (ph.fast == 1 || ph.fast == 3) {  // 3: staged, uniform masses (no per-slot mass factors)
    t.sm = nullptr;
    t.smf = nullptr;
    t.soff = reinterpret_cast<long long*>(after_v);
  } else if (ph.fast == 2) {  // streamed FAST: stencil 1/m instead of per-slot mass factors
    t.sm = nullptr;
    t.smf = after_v;
    t.soff = reinterpret_cast<long long*>(t.smf + ph.S);
  } else {
    t.sm = after_v;
    t.smf = t.sm + ph.S;
    t.soff = reinterpret_cast<long long*>(t.smf + ph.S);
  }
  t.sdiag = reinterpret_cast<double*>(t.soff + mc);
  t.sden = t.sdiag + mc;
  t.sy = t.sden + mc;
  t.spf = t.sy + mc;
  t.sqf = ph.fast == 1 ? t.spf + ph.SC + 2 : nullptr;
  t.skf = (ph.fast == 1 ? t.sqf : t.spf) + ph.SC + 2;
  t.snl = reinterpret_cast<uint16_t*>(t.skf + static_cast<size_t>(D) * ph.MR);
  return t;
}

// RN(x/d) from y = RN(1/d) (see the file comment).
__device__ __forceinline__ double div_by(double x, double d, double y) {
  const double q0 = x * y;
  const double r = __fma_rn(-d, q0, x);
  return r == 0.0 ? q0 : __fma_rn(r, y, q0);
}

template <bool ORDERED>
__device__ __forceinline__ double quot(double x, double d, double y) {
  return ORDERED ? div_by(x, d, y) : x * y;
}

#ifdef TLSPH_SWEEP_TIMING
// Debug build only: per cell task, slot 0 %globaltimer at start, slots 1-7
// clock64 at the stages of k_sweep_fast, slot 8 the particle count.
constexpr int kStampSlots = 10;
__device__ unsigned long long g_sweep_stamp[1 << 16][kStampSlots];
__device__ __forceinline__ void stamp(long long cell, int k) {
  if (threadIdx.x == 0 && cell < (1 << 16)) {
    unsigned long long t;
    if (k == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    else t = static_cast<unsigned long long>(clock64());
    g_sweep_stamp[cell][k] = t;
  }
}
#else
__device__ __forceinline__ void stamp(long long, int) {}
#endif

// ------------------------------------------------------------------ per-sweep folds
// damping.cpp:65-74: sum_b, sum_b2 in slot order, diag, denominator (its
// reciprocal feeds the corrected division on the chain).
// ORDERED: the reference's slot-order folds of b = eta G dt/2. FAST: from the
// static per-particle sums of G and G^2 (sum b = kb sum G, sum b^2 = kb^2 sum G^2,
// kb = eta dt/2; reassociation, FAST tolerance class), one read per particle.
template <bool ORDERED>
__global__ void k_sweep_folds(DFields f, double eta, double dt_fixed, int dt_from_scalars,
                              const DScalars* __restrict__ sc) {
  if (dt_from_scalars && sc->halt) return;
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= f.n) return;
  const double dt_half = 0.5 * (dt_from_scalars ? sc->dt : dt_fixed);
  double sb = 0.0, sb2 = 0.0;
  if (ORDERED) {
    const long long hi = f.offs[i + 1];
    for (long long s = f.offs[i]; s < hi; ++s) {
      const double b = eta * f.pf[s] * dt_half;
      sb = sb + b;
      sb2 = sb2 + b * b;
    }
  } else {
    const double kb = eta * dt_half;
    sb = kb * f.pfsum[i];
    sb2 = (kb * kb) * f.pfsq[i];
  }
  const double diag = sb - f.m[i];
  const double den = diag * diag + sb2;
  // a constrained particle is never updated as i (damping.cpp:151); the FAST
  // chain reads the mark from its diagonal
  f.fdiag[i] = f.flag[i] ? __longlong_as_double(0x7ff8000000000000ll) : diag;
  f.fden[i] = den;
  f.fy[i] = 1.0 / den;
}

// ------------------------------------------------------------------ per-sweep pairwise factors
// damping.cpp:91-106: b = eta G dt_pair, k = b / (m_i m_j - (m_i + m_j) b), dt_pair = dt/4 (the
// palindrome's half steps, :171-176). Velocity-independent, so formed once per (eta, dt) for every
// slot (IEEE division, the reference's operation order) and staged with the slot block.
__global__ void k_pair_factors(DFields f, double eta, double dt_fixed, int dt_from_scalars,
                               const DScalars* __restrict__ sc) {
  if (dt_from_scalars && sc->halt) return;
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= f.n) return;
  const double dt_pair = 0.5 * (0.5 * (dt_from_scalars ? sc->dt : dt_fixed));
  const double mi = f.m[i];
  const long long hi = f.offs[i + 1];
  for (long long s = f.offs[i]; s < hi; ++s) {
    const double b = eta * f.pf[s] * dt_pair;
    const double mj = f.m[f.nbr[s]];
    const double denom = mi * mj - (mi + mj) * b;
    f.pkf[s] = b / denom;
  }
}

// ------------------------------------------------------------------ staging (step 1)
template <int D>
__device__ __forceinline__ long long phase_cell(const Phase& ph, const DFields& f, long long k, int c[3]) {
  const long long lin = ph.cells[k];
  c[0] = static_cast<int>(lin % f.dims[0]);
  c[1] = static_cast<int>((lin / f.dims[0]) % f.dims[1]);
  c[2] = D == 3 ? static_cast<int>(lin / (static_cast<long long>(f.dims[0]) * f.dims[1])) : 0;
  return lin;
}

// Aligned supersets of the cell's per-particle and per-slot ranges.
struct CellSpan {
  long long p0, p1, s0, s1;
  __device__ long long o0() const { return p0 & ~1ll; }  // offs[p0..p1]
  __device__ long long o1() const { return (p1 + 2) & ~1ll; }
  __device__ long long q0() const { return p0 & ~1ll; }  // fold constants of p0..p1-1
  __device__ long long q1() const { return (p1 + 1) & ~1ll; }
  __device__ long long f0() const { return s0 & ~1ll; }  // pair factors
  __device__ long long f1() const { return (s1 + 1) & ~1ll; }
  __device__ long long n0() const { return s0 & ~7ll; }  // u16 neighbour indices
  __device__ long long n1() const { return (s1 + 7) & ~7ll; }
};

// Executed by one whole warp: padded tile layout (exclusive scan of the
// 16-byte aligned row lengths, as stencil_segments), segment table; the
// stencil rows (v, 1/m and optionally m) by per-lane 16-byte cp.async over
// the flattened row table, the cell's slot block, row offsets and fold
// constants by bulk copies on the mbarrier. MASS: also stage m (ORDERED
// divisions, pairwise).
// HDR: the bank-spread rows' per-particle headers take the place of the fold denominators (unused
// by the FAST chain).
// TROWS (no MASS): each stencil row's velocities (and, without QF, its 1/m) by one bulk copy per
// component (lane q < 3^(D-1) issues row q's) on the same mbarrier, instead of per-lane 16-byte
// cp.async over the flattened row table -- no per-pair address arithmetic (~1,000 instructions
// per cell) and no LSU wavefronts for the shared-memory writes.
#ifndef TLSPH_SWEEP_TROWS
#define TLSPH_SWEEP_TROWS 1
#endif
template <int D, bool FOLD, bool MASS, bool PDL = false, bool QF = false, bool SLOTS = true, bool UNI = false,
          bool HDR = false, bool TROWS = false>
__device__ __forceinline__ void issue_staging(const DFields& f, const Tile<D>& t, const CellSpan& cs,
                                              long long sstart, long long send, int lane,
                                              const uint16_t* nl_src = nullptr, const double* pf_src = nullptr) {
  constexpr int kSegs = seg_count<D>();
  const int slen = static_cast<int>(send - sstart);
  const int par = static_cast<int>(sstart & 1);
  const int plen = slen > 0 ? ((slen + par + 1) & ~1) : 0;
  int incl = plen;
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const int x = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += x;
  }
  const int sbase = incl - plen + par;
  if (lane < kSegs) {
    t.seg_start[lane] = sstart;
    t.seg_len[lane] = slen;
    t.seg_base[lane] = sbase;
  }
  uint32_t mybytes = 0;
  if (lane == 0) mybytes = static_cast<uint32_t>((cs.o1() - cs.o0()) * 8);
  else if (SLOTS && lane == 1) mybytes = static_cast<uint32_t>((cs.f1() - cs.f0()) * 8);
  else if (SLOTS && lane == 2) mybytes = static_cast<uint32_t>((cs.n1() - cs.n0()) * 2);
  else if (FOLD && lane == 3) mybytes = static_cast<uint32_t>((cs.q1() - cs.q0()) * 8 * 3);
  else if (SLOTS && QF && !UNI && lane == 4) mybytes = static_cast<uint32_t>((cs.f1() - cs.f0()) * 8);
  uint32_t total = mybytes;
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) total += __shfl_xor_sync(kFull, total, o);
  static_assert(!TROWS || !MASS, "bulk row copies stage the velocities and, without QF, the stencil's 1/m");
  if (lane == 0) {
    mbar_init(t.bar, TROWS ? 2 : 1);  // TROWS: the static data and the rows arrive separately
    fence_proxy_async_smem();  // the initialised barrier is visible to the TMA unit
    mbar_arrive_expect_tx(t.bar, total);
  }
  __syncwarp();
  stamp(blockIdx.x, 9);
  if (lane == 0) {
    tma_load_1d(t.soff, f.offs + cs.o0(), mybytes, t.bar);
  } else if (SLOTS && lane == 1) {
    tma_load_1d(t.spf, (pf_src ? pf_src : f.pf) + cs.f0(), mybytes, t.bar);
  } else if (SLOTS && lane == 2) {
    tma_load_1d(t.snl, (nl_src ? nl_src : f.nloc) + cs.n0(), mybytes, t.bar);
  } else if (FOLD && lane == 3) {
    const uint32_t nb = static_cast<uint32_t>((cs.q1() - cs.q0()) * 8);
    tma_load_1d(t.sdiag, f.fdiag + cs.q0(), nb, t.bar);
    if (HDR) tma_load_1d(t.sden, f.ghdr + cs.q0(), nb, t.bar);
    else tma_load_1d(t.sden, f.fden + cs.q0(), nb, t.bar);
    tma_load_1d(t.sy, f.fy + cs.q0(), nb, t.bar);
  } else if (SLOTS && QF && !UNI && lane == 4) {
    tma_load_1d(t.sqf, f.qf + cs.f0(), mybytes, t.bar);
  }
#ifndef TLSPH_STREAM_L2PF
#define TLSPH_STREAM_L2PF 1
#endif
  if (!SLOTS && TLSPH_STREAM_L2PF) {  // streamed slot block: bring it into L2 ahead of the chain's register loads
    if (lane == 1)
      tma_prefetch_l2_stream((pf_src ? pf_src : f.pf) + cs.f0(), static_cast<uint32_t>((cs.f1() - cs.f0()) * 8));
    else if (lane == 2)
      tma_prefetch_l2_stream((nl_src ? nl_src : f.nloc) + cs.n0(), static_cast<uint32_t>((cs.n1() - cs.n0()) * 2));
  }
  stamp(blockIdx.x, 3);
  constexpr int center = D == 2 ? 1 : 4;
  if (TROWS) {
    const uint32_t row_bytes = lane < kSegs ? static_cast<uint32_t>(plen) * 8u : 0u;
    uint32_t rows_total = row_bytes;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) rows_total += __shfl_xor_sync(kFull, rows_total, o);  // lanes 0-15 hold the rows
    const int lbase_t =
        __shfl_sync(kFull, sbase, center) + static_cast<int>(cs.p0 - __shfl_sync(kFull, sstart, center));
    if (lane == 0) reinterpret_cast<int*>(t.bar + 1)[0] = lbase_t;
    if (PDL) grid_dependency_wait();  // the velocities are written by the preceding phase
    if (lane == 0) mbar_arrive_expect_tx(t.bar, rows_total * (QF ? D : D + 1));
    __syncwarp();
    if (row_bytes) {
      const long long g = sstart - par;
      const int tb = sbase - par;
#pragma unroll
      for (int d = 0; d < D; ++d) tma_load_1d(t.sv[d] + tb, f.v[d] + g, row_bytes, t.bar);
      if (!QF) tma_load_1d(t.smf + tb, f.minvf + g, row_bytes, t.bar);
    }
    return;
  }
  const RowPairs rp = row_pairs(sstart, lane < kSegs ? slen : 0, sbase, lane);
  auto copy_pair = [&](long long g, int tt) {
#pragma unroll
    for (int d = 0; d < D; ++d) cp_async16(t.sv[d] + tt, f.v[d] + g);
    if (!QF) cp_async16(t.smf + tt, f.minvf + g);
    if (MASS) cp_async16(t.sm + tt, f.m + g);
  };
  // The copy addresses are static: with PDL they are formed before waiting for
  // the preceding phase (stencils of up to kPreIter x 32 pairs), so only the
  // copies themselves follow the wait.
  constexpr int kPreIter = 16;
  if (PDL && rp.total <= kPreIter * kWarp) {
    long long gp[kPreIter];
    int tp[kPreIter];
#pragma unroll
    for (int it = 0; it < kPreIter; ++it) {
      gp[it] = -1;
      tp[it] = 0;
      if (it * kWarp < rp.total) {  // warp-uniform
        const int p = it * kWarp + lane;
        int q, off;
        locate_pair<D>(rp, p, q, off);
        const long long g = 2 * (__shfl_sync(kFull, rp.gp, q) + off);
        const int tt = 2 * (__shfl_sync(kFull, rp.tp, q) + off);
        if (p < rp.total) {
          gp[it] = g;
          tp[it] = tt;
        }
      }
    }
    grid_dependency_wait();  // the velocities are written by the preceding phase
#pragma unroll
    for (int it = 0; it < kPreIter; ++it)
      if (gp[it] >= 0) copy_pair(gp[it], tp[it]);
  } else {
    if (PDL) grid_dependency_wait();
    for (int base = 0; base < rp.total; base += kWarp) {
      const int p = base + lane;
      int q, off;
      locate_pair<D>(rp, p, q, off);
      const long long g = 2 * (__shfl_sync(kFull, rp.gp, q) + off);
      const int tt = 2 * (__shfl_sync(kFull, rp.tp, q) + off);
      if (p < rp.total) copy_pair(g, tt);
    }
  }
  const int lbase =
      __shfl_sync(kFull, sbase, center) + static_cast<int>(cs.p0 - __shfl_sync(kFull, sstart, center));
  if (lane == 0) reinterpret_cast<int*>(t.bar + 1)[0] = lbase;  // the centre row holds the cell's particles
}

// Staging complete: bulk copies landed and this thread's cp.async copies done.
template <int D>
__device__ __forceinline__ void wait_staging(const Tile<D>& t) {
  cp_async_wait_all();
  mbar_wait(t.bar, 0);
}

// Write the staged stencil rows back to v; one warp per call. Lane q < 3^(D-1)
// writes the 16-byte aligned interior of row q with one bulk store per
// component; ragged row ends (odd first or last element) by plain stores.
template <int D>
__device__ __forceinline__ void writeback_rows(const DFields& f, const Tile<D>& t, int lane) {
  constexpr int kSegs = seg_count<D>();
#ifdef TLSPH_WB_PLAIN
  __syncwarp();
#pragma unroll 1
  for (int q = 0; q < kSegs; ++q) {
    const long long rs = t.seg_start[q];
    const int len = t.seg_len[q], tb = t.seg_base[q];
    for (int e = lane; e < len; e += 32) {
#pragma unroll
      for (int d = 0; d < D; ++d) f.v[d][rs + e] = t.sv[d][tb + e];
    }
  }
  return;
#endif
  fence_proxy_async_smem();  // the chain's shared-memory writes, visible to the bulk copies
  __syncwarp();
  if (lane < kSegs) {
    const long long rs = t.seg_start[lane];
    const int len = t.seg_len[lane];
    const int tb = t.seg_base[lane];
    if (len > 0) {
      const long long re = rs + len;
      const long long a0 = (rs + 1) & ~1ll, a1 = re & ~1ll;  // aligned interior [a0, a1)
      const int ta = tb + static_cast<int>(a0 - rs);
      if (a1 > a0) {
#pragma unroll
        for (int d = 0; d < D; ++d)
          tma_store_1d(f.v[d] + a0, t.sv[d] + ta, static_cast<uint32_t>((a1 - a0) * 8));
      }
      if (rs & 1) {
#pragma unroll
        for (int d = 0; d < D; ++d) f.v[d][rs] = t.sv[d][tb];
      }
      if ((re & 1) && re - 1 >= a0) {
#pragma unroll
        for (int d = 0; d < D; ++d) f.v[d][re - 1] = t.sv[d][tb + len - 1];
      }
      bulk_commit();
      bulk_wait_read();  // the tile must outlive the copies' reads
    }
  }
}

// Fused halo exchange of a slab: a cell task whose stencil
// reaches a column shared with a neighbouring slab also stores those particles'
// new velocities straight into the peer's arrays (over NVLink when the peer is
// another GPU). Same-phase stencils are disjoint, so the peer does not write
// these particles in this phase and reads them only after the phase barrier.
template <int D>
__device__ __forceinline__ void writeback_peers(const DFields& f, const Tile<D>& t, const int c[3], int tid,
                                                int nthreads) {
  if (!f.peer_idx) return;
  const bool near = (f.peer_x[0] >= 0 && c[0] - 1 <= f.peer_x[0] + 1) ||
                    (f.peer_x[1] >= 0 && c[0] + 1 >= f.peer_x[1] - 1);  // uniform per cell
  if (!near) return;
  constexpr int kSegs = seg_count<D>();
  for (int q = 0; q < kSegs; ++q) {
    const long long g0 = t.seg_start[q];
    const int b = t.seg_base[q], len = t.seg_len[q];
    for (int e = tid; e < len; e += nthreads) {
      const int pi = f.peer_idx[g0 + e];
      if (pi == -1) continue;
      const int side = pi >= 0 ? 1 : 0;
      const int idx = pi >= 0 ? pi : -2 - pi;
#pragma unroll
      for (int d = 0; d < D; ++d) f.peer_v[side][d][idx] = t.sv[d][b + e];
    }
  }
}

// ------------------------------------------------------------------ colour phase
// K > 0: rows up to 32 K slots run the branch-free register path; K = 0: generic loop only.
template <int D, int SCHEME, bool ORDERED, int K>
__global__ void __launch_bounds__(32 * D)
k_sweep_phase(DFields f, Phase ph, const DScalars* __restrict__ sc) {
  if (ph.dt_from_scalars && sc->halt) return;
  grid_launch_dependents();  // PDL: the next phase stages its static data while this one runs
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x;
  const int warp = tid / kWarp, lane = tid % kWarp;
  const long long k = blockIdx.x;
  int c[3];
  const long long lin = phase_cell<D>(ph, f, k, c);
  constexpr int kSegs = seg_count<D>();
  Tile<D> t = carve<D>(smem, ph);
  const double dt = ph.dt_from_scalars ? sc->dt : ph.dt;
  const double dt_half = 0.5 * dt;
  const double dt_op = SCHEME == TLSPH_SCHEME_PARTICLE_SPLIT ? dt_half : 0.5 * dt_half;  // pair step dt/4
  const double eta = ph.eta;

  // ---- 1. staging. All index loads are issued before any of them is used.
  CellSpan cs{f.cell_start[lin], f.cell_start[lin + 1], f.cell_slot[lin], f.cell_slot[lin + 1]};
  long long sstart = 0, send = 0;
  if (warp == 0) locate_row<D>(f, c, lane, sstart, send);
  if (cs.p0 == cs.p1) return;  // empty cell (uniform across the CTA)
  const long long p0 = cs.p0, p1 = cs.p1, s0 = cs.s0;
  const int np = static_cast<int>(p1 - p0);
  if (warp == 0) issue_staging<D, SCHEME == TLSPH_SCHEME_PARTICLE_SPLIT, true, true>(f, t, cs, sstart, send, lane);
  if (warp == 0) cp_async_wait_all();
  __syncthreads();  // barrier initialised and row copies landed before anyone waits on it
  mbar_wait(t.bar, 0);
  const int lbase = reinterpret_cast<const int*>(t.bar + 1)[0];
  const long long* offc = t.soff + (p0 - cs.o0());  // offc[k] = offs[p0 + k]
  const double* pfc = t.spf + (s0 - cs.f0());
  const uint16_t* nlc = t.snl + (s0 - cs.n0());
  const double* fdg = t.sdiag + (p0 - cs.q0());
  const double* fdn = t.sden + (p0 - cs.q0());
  const double* fyy = t.sy + (p0 - cs.q0());

  // ---- 2. the chain: warp d owns velocity component d
  if (warp < D) {
    double* const vd = t.sv[0] + static_cast<size_t>(warp) * ph.S;
    static_assert(SCHEME == TLSPH_SCHEME_PARTICLE_SPLIT, "pairwise split: k_sweep_pairwise");
    {
      constexpr int KK = K > 0 ? K : 1;
      // metadata of the next particle in chain order; none of it depends on the chain
      int pk_n = ph.forward ? 0 : np - 1;
      int lo_n = static_cast<int>(offc[pk_n] - s0), cnt_n = static_cast<int>(offc[pk_n + 1] - s0) - lo_n;
      int jq_n[KK];
      bool up_n[KK];
      double b_n[KK], bm_n[KK];
      auto meta = [&](int lo_, int cnt_, int li_, int* jq, bool* up, double* b, double* bm) {
#pragma unroll
        for (int u = 0; u < KK; ++u) {
          const int s = lane + u * kWarp;
          const bool v = s < cnt_;
          const int j = v ? nlc[lo_ + s] : li_;  // invalid lanes point at i itself with b = 0
          const double mf = t.smf[j];
          jq[u] = j;
          up[u] = v && mf > 0.0;  // clamped j: writes discarded (damping.cpp:84-86)
          b[u] = v ? eta * pfc[lo_ + s] * dt_op : 0.0;
          bm[u] = up[u] ? quot<ORDERED>(b[u], t.sm[j], mf) : 0.0;
        }
      };
      meta(lo_n, cnt_n, lbase + pk_n, jq_n, up_n, b_n, bm_n);
      for (int kk = 0; kk < np; ++kk) {
        const int pk = pk_n, lo = lo_n, cnt = cnt_n;
        int jq[KK];
        bool up[KK];
        double bq[KK], bmq[KK];
#pragma unroll
        for (int u = 0; u < KK; ++u) {
          jq[u] = jq_n[u];
          up[u] = up_n[u];
          bq[u] = b_n[u];
          bmq[u] = bm_n[u];
        }
        if (kk + 1 < np) {  // next particle's metadata, off the chain
          pk_n = ph.forward ? kk + 1 : np - 2 - kk;
          lo_n = static_cast<int>(offc[pk_n] - s0);
          cnt_n = static_cast<int>(offc[pk_n + 1] - s0) - lo_n;
          meta(lo_n, cnt_n, lbase + pk_n, jq_n, up_n, b_n, bm_n);
        }
        const int li = lbase + pk;
        if (t.smf[li] < 0.0 || cnt == 0) continue;  // constrained i (damping.cpp:151) / no neighbours (:54)
        const double diag = fdg[pk], den = fdn[pk], y = fyy[pk];
        const double vi = vd[li];
        double R = 0.0;
        double rate, vnew;
        if (K > 0 && cnt <= K * kWarp) {
          double vq[KK];
#pragma unroll
          for (int u = 0; u < KK; ++u) vq[u] = vd[jq[u]];
          if (ORDERED) {
            // every lane forms its slots' terms b (v_i - v_j) exactly as the reference does;
            // lane 0 folds them in slot order (damping.cpp:65-71) from the warp's scratch
            double* const term = t.skf + static_cast<size_t>(warp) * ph.MR;
#pragma unroll
            for (int u = 0; u < KK; ++u)
              if (lane + u * kWarp < cnt) term[lane + u * kWarp] = bq[u] * (vi - vq[u]);
            __syncwarp();
            if (lane == 0) {
              int s = 0;
#pragma unroll 4
              for (; s + 1 < cnt; s += 2) {
                const double2 tt = *reinterpret_cast<const double2*>(term + s);
                R = R - tt.x;
                R = R - tt.y;
              }
              if (s < cnt) R = R - term[s];
            }
            R = __shfl_sync(kFull, R, 0);
          } else {
            double r = 0.0;
#pragma unroll
            for (int u = 0; u < KK; ++u) r = r - bq[u] * (vi - vq[u]);
            R = warp_sum(r);
          }
          rate = quot<ORDERED>(R, den, y);
          vnew = vi + diag * rate;
#pragma unroll
          for (int u = 0; u < KK; ++u) {
            const double pred = vq[u] - bq[u] * rate;
            const double nv = vq[u] - bmq[u] * (vnew - pred);
            if (up[u]) vd[jq[u]] = nv;
          }
        } else {
          // long rows (irregular bodies): strided loop
          if (ORDERED) {
            if (lane == 0) {
              for (int s = lo; s < lo + cnt; ++s) {
                const double b = eta * pfc[s] * dt_op;
                R = R - b * (vi - vd[nlc[s]]);
              }
            }
            R = __shfl_sync(kFull, R, 0);
          } else {
            double r = 0.0;
            for (int s = lo + lane; s < lo + cnt; s += kWarp) {
              const double b = eta * pfc[s] * dt_op;
              r = r - b * (vi - vd[nlc[s]]);
            }
            R = warp_sum(r);
          }
          rate = quot<ORDERED>(R, den, y);
          vnew = vi + diag * rate;
          __syncwarp();
          for (int s = lo + lane; s < lo + cnt; s += kWarp) {
            const int j = nlc[s];
            const double mf = t.smf[j];
            if (mf > 0.0) {
              const double b = eta * pfc[s] * dt_op;
              const double bm = quot<ORDERED>(b, t.sm[j], mf);
              const double vj = vd[j];
              const double pred = vj - b * rate;
              vd[j] = vj - bm * (vnew - pred);
            }
          }
        }
        // i is not its own neighbour, so this store cannot race the scatter above
        if (lane == 0) vd[li] = vnew;
        __syncwarp();
      }
    }
  }
  __syncthreads();

  // ---- 3. write the stencil back (rows from the tile's segment table)
  for (int q = 0; q < kSegs; ++q) {
    const long long g0 = t.seg_start[q];
    const int b = t.seg_base[q], len = t.seg_len[q];
    for (int e = tid; e < len; e += 32 * D) {
#pragma unroll
      for (int d = 0; d < D; ++d) f.v[d][g0 + e] = t.sv[d][b + e];
    }
  }
  writeback_peers<D>(f, t, c, tid, 32 * D);
}

// ------------------------------------------------------------------ FAST particle split, one warp per cell
// The whole chain of a cell in one warp (sweep_chain.cuh): every slot's
// metadata is read once for all D components and the D residuals share one
// shuffle tree.
// STREAM: the slot block is not staged; the chain reads pair factors, mass
// factors and stencil indices from global memory (L2), a particle ahead. The
// tile shrinks to the stencil velocities and per-particle constants, so many
// more cells share an SM -- the form for colours with more cells than one
// wave of staged tiles holds (large bodies).
// UNI (with STREAM, uniform masses): no stencil 1/m staged (fast_chain_stream).
// One cell task of a FAST particle-split phase, executed by one warp: staging, chain, write-back.
// PDL: the phase was launched with programmatic dependent launch (wait for the previous phase
// before the velocity copies).
template <int D, int K, bool STREAM, bool UNI, bool PDL>
__device__ __forceinline__ void fast_task(const DFields& f, const Phase& ph, long long lin, const int c[3],
                                          const Tile<D>& t, double kb, int lane) {
  const CellSpan cs{f.cell_start[lin], f.cell_start[lin + 1], f.cell_slot[lin], f.cell_slot[lin + 1]};
  long long sstart, send;
  locate_row<D>(f, c, lane, sstart, send);
  if (cs.p0 == cs.p1) return;
  stamp(blockIdx.x, 2);
  constexpr bool SPREAD = UNI && TLSPH_SWEEP_SPREAD;  // bank-spread slot rows (state.cu k_spread_rows)
  const double* const pf_rows = SPREAD ? f.pfsp : f.pf;
  // dense rows (large bodies): the streamed chain reads row p at p * dense_r; the staging call below
  // then prefetches that block (its slot range is only used for the L2 prefetch when nothing is staged)
  const bool dense = STREAM && SPREAD && f.nld != nullptr;
  const CellSpan cst = dense ? CellSpan{cs.p0, cs.p1, cs.p0 * f.dense_r, cs.p1 * f.dense_r} : cs;
  // bulk row copies for the streamed (large-body) form only: with a handful of cells per SM the
  // serialised bulk issue costs the latency-bound chain more than it saves (cfg2 0.635 -> 0.684 ms)
  issue_staging<D, true, false, PDL, !STREAM || UNI, !STREAM, UNI, SPREAD, STREAM && TLSPH_SWEEP_TROWS>(
      f, t, cst, sstart, send, lane, dense ? f.nld : UNI ? f.nlocf : f.nloc, dense ? f.pfd : pf_rows);
  stamp(blockIdx.x, 4);
  wait_staging(t);
  __syncwarp();
  stamp(blockIdx.x, 5);
  ChainTile<D> ct;
#pragma unroll
  for (int d = 0; d < D; ++d) ct.sv[d] = t.sv[d];
  ct.smf = t.smf;
  if (STREAM) {
    ct.pf = pf_rows + cs.s0;
    ct.pfb = pf_rows;
    ct.nlb = UNI ? f.nlocf : f.nloc;
    ct.s0u = static_cast<unsigned>(cs.s0);
    ct.qf = nullptr;  // formed from 1/m (fast_chain_stream)
    ct.nl = (UNI ? f.nlocf : f.nloc) + cs.s0;
    ct.minv = f.minv_uniform;
    if (dense) {
      ct.pf = f.pfd + cs.p0 * f.dense_r;
      ct.nl = f.nld + cs.p0 * f.dense_r;
    }
  } else {
    ct.pf = t.spf + (cs.s0 - cs.f0());
    ct.qf = UNI ? nullptr : t.sqf + (cs.s0 - cs.f0());
    ct.nl = t.snl + (cs.s0 - cs.n0());
    ct.minv = f.minv_uniform;
  }
  ct.offs = t.soff + (cs.p0 - cs.o0());
  ct.hdr = reinterpret_cast<const unsigned long long*>(t.sden) + (cs.p0 - cs.q0());
  ct.s0 = cs.s0;
  ct.diag = t.sdiag + (cs.p0 - cs.q0());
  ct.y = t.sy + (cs.p0 - cs.q0());
  ct.lbase = reinterpret_cast<const int*>(t.bar + 1)[0];
  ct.np = static_cast<int>(cs.p1 - cs.p0);
  ct.forward = ph.forward;
  ct.kb = kb;
  if (STREAM && SPREAD && dense) fast_chain_stream<D, K, UNI, SPREAD, STREAM && SPREAD>(ct, lane);
  else if (STREAM) fast_chain_stream<D, K, UNI, SPREAD>(ct, lane);
  else fast_chain<D, K, true, true, UNI, SPREAD>(ct, lane);
  __syncwarp();
  stamp(blockIdx.x, 6);

  writeback_peers<D>(f, t, c, lane, kWarp);
  writeback_rows<D>(f, t, lane);
  stamp(blockIdx.x, 7);
#ifdef TLSPH_SWEEP_TIMING
  if (lane == 0 && blockIdx.x < (1 << 16)) g_sweep_stamp[blockIdx.x][8] = static_cast<unsigned long long>(cs.p1 - cs.p0);
#endif
}

template <int D>
__device__ __forceinline__ void cell_coords(const DFields& f, long long lin, int c[3]) {
  c[0] = static_cast<int>(lin % f.dims[0]);
  c[1] = static_cast<int>((lin / f.dims[0]) % f.dims[1]);
  c[2] = D == 3 ? static_cast<int>(lin / (static_cast<long long>(f.dims[0]) * f.dims[1])) : 0;
}

// The whole chain of a cell in one warp (sweep_chain.cuh): every slot's
// metadata is read once for all D components and the D residuals share one
// shuffle tree.
// STREAM: the slot block is not staged; the chain reads pair factors, mass
// factors and stencil indices from global memory (L2), a particle ahead. The
// tile shrinks to the stencil velocities and per-particle constants, so many
// more cells share an SM -- the form for colours with more cells than one
// wave of staged tiles holds (large bodies).
// UNI (with STREAM, uniform masses): no stencil 1/m staged (fast_chain_stream).
// TLSPH_SWEEP_FAST_MINB (A/B): minimum resident one-warp CTAs per SM (a register bound of
// 65536 / (32 MINB)); 0: the compiler's choice
#ifndef TLSPH_SWEEP_FAST_MINB
#define TLSPH_SWEEP_FAST_MINB 0
#endif
#if TLSPH_SWEEP_FAST_MINB > 0
#define SWEEP_FAST_BOUNDS __launch_bounds__(kWarp, TLSPH_SWEEP_FAST_MINB)
#else
#define SWEEP_FAST_BOUNDS __launch_bounds__(kWarp)
#endif
template <int D, int K, bool STREAM, bool UNI>
__global__ void SWEEP_FAST_BOUNDS
k_sweep_fast(DFields f, Phase ph, const DScalars* __restrict__ sc) {
  if (ph.dt_from_scalars && sc->halt) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x;
  stamp(blockIdx.x, 0);
  stamp(blockIdx.x, 1);
  grid_launch_dependents();  // the next phase may stage its static data while this one runs
  int c[3];
  const long long lin = phase_cell<D>(ph, f, blockIdx.x, c);
  Tile<D> t = carve<D>(smem, ph);
  const double dt = ph.dt_from_scalars ? sc->dt : ph.dt;
  fast_task<D, K, STREAM, UNI, true>(f, ph, lin, c, t, ph.eta * (0.5 * dt), lane);  // b = kb * pair_factor
}

// ------------------------------------------------------------------ the dataflow sweep
// A whole FAST particle-split sweep in one persistent launch (sweep_flow below): warps dequeue
// cell tasks (cell, global phase) in the temporally blocked order and run each once the tasks it
// depends on are complete. A task touches its cell's 3^D stencil, x-1..x+1, so it depends exactly
// on the earlier-phase tasks in columns x-2..x+2; per column a counter of completed tasks, and
// pref[p][x] = the number of tasks of phases < p in column x. A column's counter reaches pref[p][x]
// only once all of those tasks are done (a task never completes before the earlier-phase tasks of
// its own column), so waiting for counter >= pref on the five columns orders every pair of
// overlapping tasks as the phase-by-phase sweep does: bitwise the same result, with no launch
// boundaries and each chunk's velocities reused from L2 across its k phases. The queue order is a
// topological order of these dependencies and every dequeued task is held by a resident warp,
// so the waits always end.
struct Flow {
  const int2* queue;  // (cell, phase) in schedule order
  long long ntask;
  const int* pref;    // (2 nb + 1) x dims[0]
  int* done;          // per column, zeroed per sweep
  unsigned long long* head;  // dequeue counter, zeroed per sweep
  int nb;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

#ifndef TLSPH_FLOW_MINB
#define TLSPH_FLOW_MINB 15
#endif
template <int D, int K, bool STREAM, bool UNI>
__global__ void __launch_bounds__(kWarp, TLSPH_FLOW_MINB)
k_sweep_flow(DFields f, Phase ph, Flow fl, const DScalars* __restrict__ sc) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x;
  grid_dependency_wait();  // fold constants, dt, the preceding step
  if (ph.dt_from_scalars && sc->halt) return;
  Tile<D> t = carve<D>(smem, ph);
  const double dt = ph.dt_from_scalars ? sc->dt : ph.dt;
  const double kb = ph.eta * (0.5 * dt);
  const int nx = f.dims[0];
  for (;;) {
    unsigned long long k = 0;
    if (lane == 0) k = atomicAdd(fl.head, 1ull);
    k = __shfl_sync(kFull, k, 0);
    if (static_cast<long long>(k) >= fl.ntask) break;
    const int2 task = fl.queue[k];
    int c[3];
    cell_coords<D>(f, task.x, c);
    if (lane < 5) {
      const int x = c[0] - 2 + lane;
      if (x >= 0 && x < nx) {
        const int need = fl.pref[static_cast<size_t>(task.y) * nx + x];
        // bounded: a schedule fault aborts the launch (~10 s) instead of hanging the device
        for (long long spin = 0; ld_acquire(fl.done + x) < need; ++spin) {
          if (spin > (1ll << 27)) __trap();
          __nanosleep(64);
        }
      }
    }
    __syncwarp();
    Phase pt = ph;
    pt.forward = task.y < fl.nb;
    fast_task<D, K, STREAM, UNI, false>(f, pt, task.x, c, t, kb, lane);
    if (lane == 0) mbar_inval(t.bar);
    bulk_wait_all();  // this lane's bulk stores performed, not only read from shared memory
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      atomicAdd(fl.done + c[0], 1);
    }
  }
}

// ------------------------------------------------------------------ pairwise split, one warp per cell
// damping.cpp:91-106 (pairwise_split_update) in the palindromic order of :171-176: per particle
// i, its slots ascending then descending, each a 2x2 implicit solve at dt/4 that changes v_i and
// v_j. The chain of a particle is carried by v_i alone (a row's j are distinct).
//   ORDERED: lanes 0..D-1 run the D components' chains in lockstep, pair after pair, in the
//            reference's operation order (bit-exact); operands of kPairBatch pairs are loaded
//            ahead of their solves.
//   FAST:    the chain is an affine recurrence in v_i: v_i <- (1 + c_s) v_i - c_s v_j,s with
//            c_s = m_j k_s, so each leg is a warp scan of affine maps (lane l owns slots
//            l K .. l K + K - 1; shuffle-up scan forward, shuffle-down scan on the reverse leg)
//            that yields v_i before every pair at once; the v_j updates
//            v_j -= m_i k_s (v_i,before - v_j) then run in parallel. Reassociated (FAST class).
// Per-slot factors k_s come precomputed (k_pair_factors) in the staged slot block.
template <int D>
__device__ __forceinline__ void affine_compose(double& A, double (&B)[D], double A2, const double (&B2)[D]) {
  // (A, B) <- (A, B) o (A2, B2): x -> A (A2 x + B2) + B
#pragma unroll
  for (int d = 0; d < D; ++d) B[d] = __fma_rn(A, B2[d], B[d]);
  A = A * A2;
}

template <int D, int K, bool ORDERED>
__global__ void __launch_bounds__(kWarp)
k_sweep_pairwise(DFields f, Phase ph, const DScalars* __restrict__ sc) {
  if (ph.dt_from_scalars && sc->halt) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x;
  grid_launch_dependents();
  int c[3];
  const long long lin = phase_cell<D>(ph, f, blockIdx.x, c);
  Tile<D> t = carve<D>(smem, ph);
  const CellSpan cs{f.cell_start[lin], f.cell_start[lin + 1], f.cell_slot[lin], f.cell_slot[lin + 1]};
  long long sstart, send;
  locate_row<D>(f, c, lane, sstart, send);
  if (cs.p0 == cs.p1) return;
  issue_staging<D, false, true, true>(f, t, cs, sstart, send, lane, nullptr, f.pkf);
  wait_staging(t);
  __syncwarp();
  const int lbase = reinterpret_cast<const int*>(t.bar + 1)[0];
  const long long* offc = t.soff + (cs.p0 - cs.o0());
  const double* kfc = t.spf + (cs.s0 - cs.f0());  // staged pairwise factors
  const uint16_t* nlc = t.snl + (cs.s0 - cs.n0());
  const int np = static_cast<int>(cs.p1 - cs.p0);

  for (int kk = 0; kk < np; ++kk) {
    const int pk = ph.forward ? kk : np - 1 - kk;
    const int li = lbase + pk;
    if (t.smf[li] < 0.0) continue;  // constrained i (damping.cpp:151)
    const int lo = static_cast<int>(offc[pk] - cs.s0), cnt = static_cast<int>(offc[pk + 1] - cs.s0) - lo;
    if (cnt == 0) continue;
    const double mi = t.sm[li];
    if (ORDERED || K == 0 || cnt > K * kWarp) {
      if (lane < D) {
        double* const vd = t.sv[0] + static_cast<size_t>(lane) * ph.S;  // component arrays are contiguous
        constexpr int kPairBatch = 8;
        double vi = vd[li];
        for (int pass = 0; pass < 2; ++pass) {
          for (int u0 = 0; u0 < cnt; u0 += kPairBatch) {
            int jb[kPairBatch];
            double kfb[kPairBatch], mjb[kPairBatch], vjb[kPairBatch];
            bool upb[kPairBatch];
#pragma unroll
            for (int q = 0; q < kPairBatch; ++q) {
              const int u = u0 + q < cnt ? u0 + q : cnt - 1;
              const int s = pass == 0 ? u : cnt - 1 - u;
              const int j = nlc[lo + s];
              jb[q] = j;
              kfb[q] = kfc[lo + s];
              mjb[q] = t.sm[j];
              vjb[q] = vd[j];
              upb[q] = t.smf[j] > 0.0;
            }
#pragma unroll
            for (int q = 0; q < kPairBatch; ++q) {
              if (u0 + q < cnt) {
                const double scaled = kfb[q] * (vi - vjb[q]);
                vi = vi + mjb[q] * scaled;
                if (upb[q]) vd[jb[q]] = vjb[q] - mi * scaled;  // clamped j: discarded (damping.cpp:105)
              }
            }
          }
        }
        vd[li] = vi;
      }
    } else {
      constexpr int KK = K > 0 ? K : 1;
      int jq[KK];
      bool up[KK];
      double kq[KK], al[KK], vj[KK][D], vi0[D];
#pragma unroll
      for (int d = 0; d < D; ++d) vi0[d] = t.sv[d][li];
#pragma unroll
      for (int u = 0; u < KK; ++u) {
        const int s = lane * KK + u;
        const bool v = s < cnt;
        const int j = v ? nlc[lo + s] : li;
        jq[u] = j;
        kq[u] = v ? kfc[lo + s] : 0.0;
        up[u] = v && t.smf[j] > 0.0;
        al[u] = v ? t.sm[j] * kq[u] : 0.0;  // c_s = m_j k_s (identity map for padding slots)
#pragma unroll
        for (int d = 0; d < D; ++d) vj[u][d] = t.sv[d][j];
      }
      double vfin[D];
#pragma unroll
      for (int d = 0; d < D; ++d) vfin[d] = vi0[d];
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        // this lane's slots as one affine map, in leg order
        double A = 1.0, B[D];
#pragma unroll
        for (int d = 0; d < D; ++d) B[d] = 0.0;
#pragma unroll
        for (int q = 0; q < KK; ++q) {
          const int u = pass == 0 ? q : KK - 1 - q;
          double Bu[D];
#pragma unroll
          for (int d = 0; d < D; ++d) Bu[d] = -al[u] * vj[u][d];
          // later map o earlier: x -> (1 + c) (A x + B) - c v_j
          double Al = 1.0 + al[u];
          double Bl[D];
#pragma unroll
          for (int d = 0; d < D; ++d) Bl[d] = Bu[d];
          affine_compose<D>(Al, Bl, A, B);
          A = Al;
#pragma unroll
          for (int d = 0; d < D; ++d) B[d] = Bl[d];
        }
        // inclusive scan over the lanes in leg order (forward: lower lanes first; reverse: higher)
#pragma unroll
        for (int o = 1; o < kWarp; o <<= 1) {
          double A2 = pass == 0 ? __shfl_up_sync(kFull, A, o) : __shfl_down_sync(kFull, A, o);
          double B2[D];
#pragma unroll
          for (int d = 0; d < D; ++d) B2[d] = pass == 0 ? __shfl_up_sync(kFull, B[d], o) : __shfl_down_sync(kFull, B[d], o);
          const bool has = pass == 0 ? lane >= o : lane + o < kWarp;
          if (has) affine_compose<D>(A, B, A2, B2);
        }
        // exclusive prefix applied to the leg's start value: v_i before this lane's first slot
        double vstart[D];
#pragma unroll
        for (int d = 0; d < D; ++d) vstart[d] = pass == 0 ? vi0[d] : vfin[d];
        double Ae = pass == 0 ? __shfl_up_sync(kFull, A, 1) : __shfl_down_sync(kFull, A, 1);
        double x[D];
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const double Be = pass == 0 ? __shfl_up_sync(kFull, B[d], 1) : __shfl_down_sync(kFull, B[d], 1);
          const bool first = pass == 0 ? lane == 0 : lane == kWarp - 1;
          x[d] = first ? vstart[d] : __fma_rn(Ae, vstart[d], Be);
        }
        // the leg's end value: the whole composition (last lane in leg order)
        const int endl = pass == 0 ? kWarp - 1 : 0;
        const double At = __shfl_sync(kFull, A, endl);
        double vend[D];
#pragma unroll
        for (int d = 0; d < D; ++d) vend[d] = __fma_rn(At, vstart[d], __shfl_sync(kFull, B[d], endl));
        // the pairs of this lane: v_j updates from v_i before each pair
#pragma unroll
        for (int q = 0; q < KK; ++q) {
          const int u = pass == 0 ? q : KK - 1 - q;
          const double mk = mi * kq[u];
#pragma unroll
          for (int d = 0; d < D; ++d) {
            const double w = x[d] - vj[u][d];
            x[d] = __fma_rn(al[u], w, x[d]);  // v_i + m_j k (v_i - v_j)
            if (up[u]) vj[u][d] = vj[u][d] - mk * w;
          }
        }
#pragma unroll
        for (int d = 0; d < D; ++d) vfin[d] = vend[d];
      }
#pragma unroll
      for (int u = 0; u < KK; ++u)
        if (up[u]) {
#pragma unroll
          for (int d = 0; d < D; ++d) t.sv[d][jq[u]] = vj[u][d];
        }
      if (lane == 0) {
#pragma unroll
        for (int d = 0; d < D; ++d) t.sv[d][li] = vfin[d];
      }
    }
    __syncwarp();
  }
  writeback_peers<D>(f, t, c, lane, kWarp);
  writeback_rows<D>(f, t, lane);
}

template <int D, int K, bool ORDERED>
void launch_pairwise(const DevSystem& s, const DFields& f, Phase ph) {
  ph.fast = 0;  // masses and 1/m staged; the slot block carries the pairwise factors
  const size_t smem = tile_bytes<D>(ph.S, ph.SC, ph.MC, 0, 0);
  ph.MR = 0;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    CK(cudaFuncSetAttribute(k_sweep_pairwise<D, K, ORDERED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(smem)));
    configured = smem;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(ph.ncol));
  cfg.blockDim = dim3(kWarp);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_sweep_pairwise<D, K, ORDERED>, f, ph, s.scal.p));
}

template <int D>
void launch_pairwise_any(const DevSystem& s, const DFields& f, const Phase& ph) {
  const int K = (s.max_row + kWarp - 1) / kWarp;
  if (s.reduction == TLSPH_REDUCTION_ORDERED || K > 4) launch_pairwise<D, 0, true>(s, f, ph);
  else if (K <= 1) launch_pairwise<D, 1, false>(s, f, ph);
  else if (K == 2) launch_pairwise<D, 2, false>(s, f, ph);
  else if (K == 3) launch_pairwise<D, 3, false>(s, f, ph);
  else launch_pairwise<D, 4, false>(s, f, ph);
}

// Staged or streamed slot block (tlsph_dev_set_sweep_tiling); AUTO: streamed
// when the colour's cells exceed two waves of staged tiles
// (TLSPH_SWEEP_STREAM=0/1 overrides AUTO, for A/B runs).
inline bool stream_slots(const DevSystem& s, const Phase& ph, size_t staged_bytes, int waves = 2) {
  if (s.sweep_tiling != TLSPH_SWEEP_TILING_AUTO) return s.sweep_tiling == TLSPH_SWEEP_TILING_STREAMED;
  static const int force = [] {
    const char* e = std::getenv("TLSPH_SWEEP_STREAM");
    return e && *e ? std::atoi(e) : -1;
  }();
  if (force >= 0) return force != 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // measured crossover: staged still wins at ~1.6 waves (cfg3: 1.133 vs 1.188 ms per sweep) and
  // loses from ~11 waves on (cfg4 12.5 vs 10.4, cfg5-weak 24.2 vs 18.0)
  const long long per_sm = std::max<long long>(1, static_cast<long long>((228 * 1024) / (staged_bytes + 1024)));
  return std::max(ph.ncol, ph.ncol_colour) > waves * per_sm * sms;
}

inline bool uniform_disabled() {  // TLSPH_SWEEP_UNIFORM=0: the stencil-1/m form even for uniform masses (A/B)
  static const bool off = [] {
    const char* e = std::getenv("TLSPH_SWEEP_UNIFORM");
    return e && *e == '0';
  }();
  return off;
}

template <int D, int K, bool STREAM, bool UNI = false>
void launch_fast_impl(const DevSystem& s, const DFields& f, Phase ph) {
  if (STREAM) {
    ph.SC = 0;  // no slot block in the tile
    ph.fast = UNI ? 1 : 2;  // stencil velocities only, or with the stencil's 1/m
  } else if (UNI) {
    ph.fast = 3;  // slot block without per-slot mass factors
  }
  size_t smem = tile_bytes<D>(ph.S, ph.SC, ph.MC, ph.MR, ph.fast);
  {
    // Spread a colour that fits in one wave over every SM: the CTA scheduler fills
    // an SM up to its resident limit, so a small tile would pack the cells onto
    // fewer SMs (more chains per scheduler, idle SMs). Pad the tile so at most
    // ceil(cells / SMs) are resident per SM.
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long per_sm = (ph.ncol + sms - 1) / sms;
    constexpr size_t kSmemSM = 228 * 1024, kReserve = 1024;
    static const int pad_mode = [] {  // TLSPH_SWEEP_PAD=0: no padding; =2: room for two phases (A/B runs)
      const char* e = std::getenv("TLSPH_SWEEP_PAD");
      return e && *e ? std::atoi(e) : 1;
    }();
    if (pad_mode && per_sm >= 1 && per_sm * pad_mode < 32) {
      const long long ps = per_sm * pad_mode;
      const size_t cap = (kSmemSM / static_cast<size_t>(ps) - kReserve) & ~static_cast<size_t>(127);
      if (cap > smem && static_cast<size_t>(ps) * (smem + kReserve) <= kSmemSM) smem = std::min<size_t>(cap, 200 * 1024);
    }
  }
  {
    // measurement knob: at most TLSPH_SWEEP_MAXCELLS cell tasks resident per SM (tile padded)
    static const int max_cells = [] {
      const char* e = std::getenv("TLSPH_SWEEP_MAXCELLS");
      return e && *e ? std::atoi(e) : 0;
    }();
    if (max_cells > 0) {
      const size_t cap = ((228 * 1024) / static_cast<size_t>(max_cells) - 1024) & ~static_cast<size_t>(127);
      if (cap > smem) smem = std::min<size_t>(cap, 200 * 1024);
    }
  }
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    CK(cudaFuncSetAttribute(k_sweep_fast<D, K, STREAM, UNI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(smem)));
    configured = smem;
  }
  // programmatic dependent launch: the phase's CTAs may start (and stage their
  // static data) while the preceding kernel finishes; they wait on it before
  // touching the velocities (griddepcontrol.wait in issue_staging)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(ph.ncol));
  cfg.blockDim = dim3(kWarp);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_sweep_fast<D, K, STREAM, UNI>, f, ph, s.scal.p));
}

template <int D, int K>
void launch_fast(const DevSystem& s, const DFields& f, const Phase& ph) {
  const bool uni = f.nlocf && !uniform_disabled();
  if (!stream_slots(s, ph, tile_bytes<D>(ph.S, ph.SC, ph.MC, ph.MR, uni ? 3 : ph.fast))) {
    if (uni) launch_fast_impl<D, K, false, true>(s, f, ph);
    else launch_fast_impl<D, K, false, false>(s, f, ph);
  } else if (f.nlocf && !uniform_disabled()) launch_fast_impl<D, K, true, true>(s, f, ph);
  else launch_fast_impl<D, K, true, false>(s, f, ph);
}

// The dataflow sweep (k_sweep_flow): one persistent launch of as many one-warp CTAs as fit.
template <int D, int K, bool STREAM, bool UNI>
void launch_flow_impl(const DevSystem& s, const DFields& f, Phase ph, const Flow& fl) {
  if (STREAM) {
    ph.SC = 0;
    ph.fast = UNI ? 1 : 2;
  } else if (UNI) {
    ph.fast = 3;
  }
  const size_t smem = tile_bytes<D>(ph.S, ph.SC, ph.MC, ph.MR, ph.fast);
  auto kern = k_sweep_flow<D, K, STREAM, UNI>;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    configured = smem;
  }
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarp, smem));
  const long long grid = std::min<long long>(static_cast<long long>(std::max(per_sm, 1)) * sms, fl.ntask);
  launch_pdl_phase(kern, static_cast<unsigned>(std::max<long long>(grid, 1)), kWarp, smem, s.stream, f, ph, fl,
                   static_cast<const DScalars*>(s.scal.p));
}

template <int D, int K>
void launch_flow(const DevSystem& s, const DFields& f, const Phase& ph, const Flow& fl) {
  const bool uni = f.nlocf && !uniform_disabled();
  if (!stream_slots(s, ph, tile_bytes<D>(ph.S, ph.SC, ph.MC, ph.MR, uni ? 3 : ph.fast))) {
    if (uni) launch_flow_impl<D, K, false, true>(s, f, ph, fl);
    else launch_flow_impl<D, K, false, false>(s, f, ph, fl);
  } else if (uni) launch_flow_impl<D, K, true, true>(s, f, ph, fl);
  else launch_flow_impl<D, K, true, false>(s, f, ph, fl);
}

// ------------------------------------------------------------------ ORDERED particle split, one warp per cell
// The bit-exact chain (damping.cpp:53-89 in the reference's operation order) with all D components
// in one warp: lanes form every slot's terms b (v_i - v_j) of every component, lane d folds
// component d's terms in slot order (the D folds run side by side), and the rate (corrected
// division), v_i and the scatter follow for all components at once. One pass over the slot
// metadata per particle instead of one per component warp (k_sweep_phase).
// STREAM (large bodies, as k_sweep_fast<STREAM>): the slot block (pair factors, stencil indices)
// is not staged but read from global memory one particle ahead (the `meta` prefetch below), after
// a bulk L2 prefetch of the cell's block; the tile shrinks to the stencil's velocities and masses,
// so about twice as many cells share an SM. Same arithmetic, same order: bit-identical.
template <int D, int K, bool STREAM = false>
__global__ void __launch_bounds__(kWarp)
k_sweep_ordered(DFields f, Phase ph, const DScalars* __restrict__ sc) {
  if (ph.dt_from_scalars && sc->halt) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x;
  grid_launch_dependents();
  int c[3];
  const long long lin = phase_cell<D>(ph, f, blockIdx.x, c);
  Tile<D> t = carve<D>(smem, ph);
  const double dt = ph.dt_from_scalars ? sc->dt : ph.dt;
  const double dt_op = 0.5 * dt;  // particle split: dt/2 (damping.cpp:133)
  const double eta = ph.eta;
  const CellSpan cs{f.cell_start[lin], f.cell_start[lin + 1], f.cell_slot[lin], f.cell_slot[lin + 1]};
  long long sstart, send;
  locate_row<D>(f, c, lane, sstart, send);
  if (cs.p0 == cs.p1) return;
  issue_staging<D, true, true, true, false, !STREAM>(f, t, cs, sstart, send, lane);
  wait_staging(t);
  __syncwarp();
  const int lbase = reinterpret_cast<const int*>(t.bar + 1)[0];
  const long long s0 = cs.s0;
  const long long* offc = t.soff + (cs.p0 - cs.o0());
  const double* pfc = STREAM ? f.pf + s0 : t.spf + (s0 - cs.f0());
  const uint16_t* nlc = STREAM ? f.nloc + s0 : t.snl + (s0 - cs.n0());
  const double* fdg = t.sdiag + (cs.p0 - cs.q0());
  const double* fdn = t.sden + (cs.p0 - cs.q0());
  const double* fyy = t.sy + (cs.p0 - cs.q0());
  const int np = static_cast<int>(cs.p1 - cs.p0);
  double* const term = t.skf;  // D x MR: component d's terms at term[d * MR + slot]

  int pk_n = ph.forward ? 0 : np - 1;
  int lo_n = static_cast<int>(offc[pk_n] - s0), cnt_n = static_cast<int>(offc[pk_n + 1] - s0) - lo_n;
  int jq_n[K];
  bool up_n[K];
  double b_n[K], bm_n[K];
  auto meta = [&](int lo_, int cnt_, int li_) {
#pragma unroll
    for (int u = 0; u < K; ++u) {
      const int sl = lane + u * kWarp;
      const bool v = sl < cnt_;
      const int j = v ? nlc[lo_ + sl] : li_;  // invalid lanes point at i itself with b = 0
      const double mf = t.smf[j];
      jq_n[u] = j;
      up_n[u] = v && mf > 0.0;  // clamped j: writes discarded (damping.cpp:84-86)
      b_n[u] = v ? eta * pfc[lo_ + sl] * dt_op : 0.0;
      bm_n[u] = up_n[u] ? div_by(b_n[u], t.sm[j], mf) : 0.0;
    }
  };
  meta(lo_n, cnt_n, lbase + pk_n);
  for (int kk = 0; kk < np; ++kk) {
    const int pk = pk_n, cnt = cnt_n;
    int jq[K];
    bool up[K];
    double bq[K], bmq[K];
#pragma unroll
    for (int u = 0; u < K; ++u) {
      jq[u] = jq_n[u];
      up[u] = up_n[u];
      bq[u] = b_n[u];
      bmq[u] = bm_n[u];
    }
    if (kk + 1 < np) {  // next particle's metadata, off the chain
      pk_n = ph.forward ? kk + 1 : np - 2 - kk;
      lo_n = static_cast<int>(offc[pk_n] - s0);
      cnt_n = static_cast<int>(offc[pk_n + 1] - s0) - lo_n;
      meta(lo_n, cnt_n, lbase + pk_n);
    }
    const int li = lbase + pk;
    if (t.smf[li] < 0.0 || cnt == 0) continue;  // constrained i (damping.cpp:151) / no neighbours (:54)
    const double diag = fdg[pk], den = fdn[pk], y = fyy[pk];
    double vi[D], vq[K][D];
#pragma unroll
    for (int d = 0; d < D; ++d) vi[d] = t.sv[d][li];
#pragma unroll
    for (int u = 0; u < K; ++u)
#pragma unroll
      for (int d = 0; d < D; ++d) vq[u][d] = t.sv[d][jq[u]];
    // terms b (v_i - v_j) exactly as the reference forms them (damping.cpp:65-71)
#pragma unroll
    for (int u = 0; u < K; ++u)
      if (lane + u * kWarp < cnt)
#pragma unroll
        for (int d = 0; d < D; ++d) term[d * ph.MR + lane + u * kWarp] = bq[u] * (vi[d] - vq[u][d]);
    __syncwarp();
    double Rl = 0.0;
    if (lane < D) {  // lane d folds component d in slot order; loads run 8 terms ahead of the adds
      const double* tc = term + lane * ph.MR;
      const double2* t2 = reinterpret_cast<const double2*>(tc);
      const int npair = cnt >> 1;
      double2 a = npair > 0 ? t2[0] : make_double2(0.0, 0.0), b = npair > 1 ? t2[1] : a;
      double2 c2 = npair > 2 ? t2[2] : a, e = npair > 3 ? t2[3] : a;
      int q = 0;
      for (; q + 4 <= npair; q += 4) {
        const double2 a1 = q + 4 < npair ? t2[q + 4] : a, b1 = q + 5 < npair ? t2[q + 5] : a;
        const double2 c1 = q + 6 < npair ? t2[q + 6] : a, e1 = q + 7 < npair ? t2[q + 7] : a;
        Rl = Rl - a.x;
        Rl = Rl - a.y;
        Rl = Rl - b.x;
        Rl = Rl - b.y;
        Rl = Rl - c2.x;
        Rl = Rl - c2.y;
        Rl = Rl - e.x;
        Rl = Rl - e.y;
        a = a1;
        b = b1;
        c2 = c1;
        e = e1;
      }
      const double2 rest[3] = {a, b, c2};
#pragma unroll
      for (int r = 0; r < 3; ++r)
        if (q + r < npair) {
          Rl = Rl - rest[r].x;
          Rl = Rl - rest[r].y;
        }
      if (cnt & 1) Rl = Rl - tc[cnt - 1];
    }
    double rate[D], vnew[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const double R = __shfl_sync(kFull, Rl, d);
      rate[d] = div_by(R, den, y);
      vnew[d] = vi[d] + diag * rate[d];
    }
#pragma unroll
    for (int u = 0; u < K; ++u)
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const double pred = vq[u][d] - bq[u] * rate[d];
        const double nv = vq[u][d] - bmq[u] * (vnew[d] - pred);
        if (up[u]) t.sv[d][jq[u]] = nv;
      }
    // i is not its own neighbour, so this store cannot race the scatter above
    if (lane == 0)
#pragma unroll
      for (int d = 0; d < D; ++d) t.sv[d][li] = vnew[d];
    __syncwarp();
  }
  writeback_peers<D>(f, t, c, lane, kWarp);
  writeback_rows<D>(f, t, lane);
}

inline bool ordered_warps() {  // TLSPH_SWEEP_ORDERED_WARPS=1: one warp per component (k_sweep_phase), A/B
  static const bool on = [] {
    const char* e = std::getenv("TLSPH_SWEEP_ORDERED_WARPS");
    return e && *e == '1';
  }();
  return on;
}

template <int D, int K>
void launch_ordered(const DevSystem& s, const DFields& f, Phase ph) {
  // large bodies: the slot block streamed from global memory (the staged / streamed choice of
  // the FAST kernel: tlsph_dev_set_sweep_tiling, AUTO beyond two waves of staged tiles)
  // (ORDERED crossover: cfg3, 3.3 waves of staged tiles, 2.87 ms staged vs 3.37 streamed; cfg4,
  // 39 waves, 38.2 vs 28.0)
  if (stream_slots(s, ph, tile_bytes<D>(ph.S, ph.SC, ph.MC, ph.MR, ph.fast), 8)) {
    ph.SC = 0;  // no slot block in the tile
    const size_t smem = tile_bytes<D>(ph.S, ph.SC, ph.MC, ph.MR, ph.fast);
    static size_t configured_s = 0;
    if (smem > 48 * 1024 && smem > configured_s) {
      CK(cudaFuncSetAttribute(k_sweep_ordered<D, K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(smem)));
      configured_s = smem;
    }
    launch_pdl_phase(k_sweep_ordered<D, K, true>, static_cast<unsigned>(ph.ncol), kWarp, smem, s.stream, f, ph,
                     s.scal.p);
    return;
  }
  const size_t smem = tile_bytes<D>(ph.S, ph.SC, ph.MC, ph.MR, ph.fast);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    CK(cudaFuncSetAttribute(k_sweep_ordered<D, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(smem)));
    configured = smem;
  }
  launch_pdl_phase(k_sweep_ordered<D, K>, static_cast<unsigned>(ph.ncol), kWarp, smem, s.stream, f, ph, s.scal.p);
}

template <int D, int SCHEME, bool ORDERED, int K>
void launch_phase(const DevSystem& s, const DFields& f, const Phase& ph) {
  const size_t smem = tile_bytes<D>(ph.S, ph.SC, ph.MC, ph.MR, ph.fast);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    CK(cudaFuncSetAttribute(k_sweep_phase<D, SCHEME, ORDERED, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(smem)));
    configured = smem;
  }
  launch_pdl_phase(k_sweep_phase<D, SCHEME, ORDERED, K>, static_cast<unsigned>(ph.ncol), 32 * D, smem, s.stream, f, ph,
                                                                                                    s.scal.p);
}

template <int D, bool ORDERED>
void launch_particle_split(const DevSystem& s, const DFields& f, const Phase& ph) {
  // slots per lane kept in registers: the smallest K that covers the longest row
  const int K = (s.max_row + kWarp - 1) / kWarp;
  if (!ORDERED && K <= 4) {
    if (K <= 1) launch_fast<D, 1>(s, f, ph);
    else if (K == 2) launch_fast<D, 2>(s, f, ph);
    else if (K == 3) launch_fast<D, 3>(s, f, ph);
    else launch_fast<D, 4>(s, f, ph);
    return;
  }
  if (ORDERED && K <= 4 && !ordered_warps()) {
    if (K <= 1) launch_ordered<D, 1>(s, f, ph);
    else if (K == 2) launch_ordered<D, 2>(s, f, ph);
    else if (K == 3) launch_ordered<D, 3>(s, f, ph);
    else launch_ordered<D, 4>(s, f, ph);
    return;
  }
  if (K <= 1) launch_phase<D, TLSPH_SCHEME_PARTICLE_SPLIT, ORDERED, 1>(s, f, ph);
  else if (K <= 2) launch_phase<D, TLSPH_SCHEME_PARTICLE_SPLIT, ORDERED, 2>(s, f, ph);
  else if (K <= 3) launch_phase<D, TLSPH_SCHEME_PARTICLE_SPLIT, ORDERED, 3>(s, f, ph);
  else if (K <= 4) launch_phase<D, TLSPH_SCHEME_PARTICLE_SPLIT, ORDERED, 4>(s, f, ph);
  else launch_phase<D, TLSPH_SCHEME_PARTICLE_SPLIT, ORDERED, 0>(s, f, ph);
}

constexpr size_t kSmemBudget = 220 * 1024;

// Shared part of a sweep's launches: tile sizes and the fold constants.
template <int D>
Phase prepare_sweep(DevSystem& s, int scheme, double eta, double dt, bool from_scal) {
  if (!s.stencil_ok)
    throw DevError(TLSPH_ERR_INVALID_ARGUMENT,
                   "damping sweep needs every neighbour inside the 3^D cell stencil (neighbors.hpp:50-52)");
  if (s.colour_start.empty()) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "damping sweep needs a neighbourhood");
  if (s.nslots >= (1ll << 32))  // the streamed chain addresses slots by 32-bit index (180 GB hold < 2^32 of them)
    throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "damping sweep: more than 2^32 - 1 neighbour slots on one device");
  const DFields f = s.fields();
  Phase ph{};
  ph.eta = eta;
  ph.dt = dt;
  ph.dt_from_scalars = from_scal ? 1 : 0;
  ph.S = (std::max(s.max_stencil, 1) + 7) & ~7;
  ph.SC = (std::max<int>(static_cast<int>(s.max_cell_slots), 1) + 7) & ~7;
  ph.MC = (std::max(s.max_cell, 1) + 1) & ~1;
  // per-warp scratch of max_row doubles: pairwise k factors, ORDERED particle-split residual terms
  ph.MR = (scheme == TLSPH_SCHEME_PAIRWISE_SPLIT || s.reduction == TLSPH_REDUCTION_ORDERED)
              ? ((std::max(s.max_row, 1) + 1) & ~1)
              : 0;
  // the single-warp FAST kernel (launch_particle_split) uses the mass-free tile
  ph.fast = scheme == TLSPH_SCHEME_PARTICLE_SPLIT && s.reduction != TLSPH_REDUCTION_ORDERED &&
            (std::max(s.max_row, 1) + kWarp - 1) / kWarp <= 4;
  const size_t per_cell = tile_bytes<D>(ph.S, ph.SC, ph.MC, ph.MR, ph.fast);
  if (per_cell > kSmemBudget)
    throw DevError(TLSPH_ERR_INVALID_ARGUMENT,
                   "damping sweep: a cell's stencil and slot block (" + std::to_string(per_cell) +
                       " bytes) exceed the shared-memory tile");
  if (scheme == TLSPH_SCHEME_PAIRWISE_SPLIT &&
      (from_scal || !s.pkf_valid || s.pkf_eta != eta || s.pkf_dt != dt)) {
    s.pkf.alloc(static_cast<size_t>(std::max<long long>(s.nslots, 1)));
    DFields fk = s.fields();
    k_pair_factors<<<static_cast<unsigned>((s.n + 127) / 128), 128, 0, s.stream>>>(fk, eta, dt, from_scal ? 1 : 0,
                                                                                   s.scal.p);
    CK_LAUNCH("k_pair_factors");
    s.pkf_valid = !from_scal;
    s.pkf_eta = eta;
    s.pkf_dt = dt;
  }
  if (scheme == TLSPH_SCHEME_PARTICLE_SPLIT) {
    // per-sweep fold constants; reused while (eta, dt) are unchanged
    const int mode = static_cast<int>(s.reduction);
    if (from_scal || !s.fold_valid || s.fold_eta != eta || s.fold_dt != dt || s.fold_mode != mode) {
      const unsigned grid = static_cast<unsigned>((s.n + 127) / 128);
      if (s.reduction == TLSPH_REDUCTION_ORDERED)
        k_sweep_folds<true><<<grid, 128, 0, s.stream>>>(f, eta, dt, from_scal ? 1 : 0, s.scal.p);
      else
        k_sweep_folds<false><<<grid, 128, 0, s.stream>>>(f, eta, dt, from_scal ? 1 : 0, s.scal.p);
      CK_LAUNCH("k_sweep_folds");
      s.fold_valid = !from_scal;
      s.fold_eta = eta;
      s.fold_dt = dt;
      s.fold_mode = mode;
    }
  }
  return ph;
}

// Colour phase `index` of pass `pass` (0: forward, colours ascending; 1:
// reverse, damping.cpp:112-121); tasks are the colour's cells whose x lies in
// the task range [task_x0, task_x1) (the whole grid unless a slab is set).
template <int D>
void launch_tasks(DevSystem& s, int scheme, Phase ph) {
  if (ph.ncol == 0) return;  // empty colour (neighbors.cpp:152) or an empty column range
  const DFields f = s.fields();
  if (scheme == TLSPH_SCHEME_PARTICLE_SPLIT) {
    if (s.reduction == TLSPH_REDUCTION_ORDERED) launch_particle_split<D, true>(s, f, ph);
    else launch_particle_split<D, false>(s, f, ph);
  } else {
    launch_pairwise_any<D>(s, f, ph);
  }
}

template <int D>
int phase_colour(int pass, int index) {
  return pass == 0 ? index : colour_count<D>() - 1 - index;
}

template <int D>
void enqueue_phase(DevSystem& s, int scheme, Phase ph, int pass, int index) {
  const int b = phase_colour<D>(pass, index);
  ph.forward = pass == 0;
  ph.cells = s.colour_cells.p + s.colour_start[b];
  ph.ncol = ph.ncol_colour = s.colour_start[b + 1] - s.colour_start[b];
  launch_tasks<D>(s, scheme, ph);
}

// Global phase p (0 .. 2 nb - 1) restricted to the tasks whose cell x lies in [xa, xb).
template <int D>
void enqueue_phase_columns(DevSystem& s, int scheme, Phase ph, int p, int xa, int xb) {
  constexpr int nb = colour_count<D>();
  const int nx = s.dims[0];
  xa = std::max(xa, 0);
  xb = std::min(xb, nx);
  if (xa >= xb) return;
  const int pass = p / nb, b = phase_colour<D>(pass, p % nb);
  const long long* st = s.xcol_start.data() + static_cast<size_t>(b) * (nx + 1);
  ph.forward = pass == 0;
  ph.cells = s.xcol_cells.p + st[xa];
  ph.ncol = st[xb] - st[xa];
  ph.ncol_colour = s.colour_start[b + 1] - s.colour_start[b];
  launch_tasks<D>(s, scheme, ph);
}

// Blocking parameters (W columns per chunk, k phases per block); {0, 0}: phase-by-phase order.
// Set by tlsph_dev_set_sweep_blocking or TLSPH_SWEEP_BLOCK="W,k" (W = 0: off). AUTO keeps the
// phase-by-phase order: measured on cfg4 / cfg5-weak the blocked schedule cuts DRAM bytes per phase
// by ~45 % (chunk velocities reused from L2) but is slower -- 14-17 ms vs 10.4 ms per cfg4 sweep
// as column-range launches (launch gaps, partial waves), 16.6 ms as the dataflow kernel (per-task
// dequeue / completion latency) -- because the phase kernel is bound by L1 traffic and chain
// latency, not by DRAM (ncu: DRAM 37 %, L1 74 % of peak; profiles/r2_sweep_blocking.md).
template <int D>
std::pair<int, int> sweep_blocking(const DevSystem& s, int scheme) {
  const int nx = s.dims[0];
  static const std::pair<int, int> forced = [] {
    const char* e = std::getenv("TLSPH_SWEEP_BLOCK");
    if (!e || !*e) return std::pair<int, int>{-1, -1};
    int w = 0, k = 0;
    if (std::sscanf(e, "%d,%d", &w, &k) < 1) return std::pair<int, int>{-1, -1};
    return std::pair<int, int>{w, k};
  }();
  if (s.task_x0 > 0 || (s.task_x1 >= 0 && s.task_x1 < nx) || s.peer_x[0] >= 0 || s.peer_x[1] >= 0 ||
      s.xcol_start.empty())
    return {0, 0};  // slabs keep the phase-by-phase order (the cross-slab protocol is per phase)
  int w = 0, k = 0;
  if (s.sweep_block_w >= 0 || forced.first >= 0) {
    w = s.sweep_block_w >= 0 ? s.sweep_block_w : forced.first;
    k = s.sweep_block_w >= 0 ? s.sweep_block_k : forced.second;
    if (k <= 0) k = w / 4;
  } else {
    return {0, 0};
  }
  if (w <= 0 || k <= 1 || w >= nx || w < 4 * k) return {0, 0};  // chunks are >= w wide (blocked_order)
  return {w, k};
}

// The temporally blocked order of one sweep's cell tasks over x-column chunks. The 2 nb phases
// are taken k at a time; within a block every chunk [lo, hi) runs its upright trapezoid (phase j
// of the block on tasks with x in [lo + 2j, hi - 2j), the sides at the body's ends not narrowed)
// and, once the chunk to its right is done, each internal chunk boundary B its inverted trapezoid
// (phase j on [B - 2j, B + 2j)). A task touches x-1..x+1, so a phase-(j+1) task depends only on
// phase-j tasks within 2 columns: every task comes after all the earlier-phase tasks it overlaps
// and before the later-phase tasks that overlap it, i.e. it sees exactly the inputs of the
// phase-by-phase order. `emit(p, xa, xb)` receives the ranges in that order.
template <int D, typename Emit>
void blocked_order(int nx, int w, int k, Emit&& emit) {
  constexpr int nphase = 2 * colour_count<D>();
  const int nchunk = std::max(1, nx / w);  // chunks of w .. 2w-1 columns: the trapezoids never invert
  std::vector<int> lo(static_cast<size_t>(nchunk) + 1);
  for (int c = 0; c <= nchunk; ++c) lo[static_cast<size_t>(c)] = static_cast<int>(static_cast<long long>(c) * nx / nchunk);
  for (int p0 = 0; p0 < nphase; p0 += k) {
    const int kk = std::min(k, nphase - p0);
    for (int c = 0; c < nchunk; ++c) {
      const int a = lo[static_cast<size_t>(c)], b = lo[static_cast<size_t>(c) + 1];
      for (int j = 0; j < kk; ++j) emit(p0 + j, a + (c > 0 ? 2 * j : 0), b - (c + 1 < nchunk ? 2 * j : 0));
      if (c > 0)
        for (int j = 1; j < kk; ++j) emit(p0 + j, a - 2 * j, a + 2 * j);
    }
  }
}

// Task queue and per-column prefix counts of the dataflow sweep for (w, k); rebuilt when they change.
template <int D>
Flow flow_schedule(DevSystem& s, int w, int k) {
  constexpr int nb = colour_count<D>();
  const int nx = s.dims[0];
  if (s.flow_w != w || s.flow_k != k || s.flow_ntask == 0) {
    std::vector<int2> q;
    q.reserve(static_cast<size_t>(s.colour_start[nb]));
    blocked_order<D>(nx, w, k, [&](int p, int xa, int xb) {
      xa = std::max(xa, 0);
      xb = std::min(xb, nx);
      if (xa >= xb) return;
      const int b = phase_colour<D>(p / nb, p % nb);
      const long long* st = s.xcol_start.data() + static_cast<size_t>(b) * (nx + 1);
      for (long long e = st[xa]; e < st[xb]; ++e) q.push_back(make_int2(s.xcol_cells_h[static_cast<size_t>(e)], p));
    });
    std::vector<int> pref(static_cast<size_t>(2 * nb + 1) * nx, 0);
    for (int p = 0; p < 2 * nb; ++p) {
      const int b = phase_colour<D>(p / nb, p % nb);
      const long long* st = s.xcol_start.data() + static_cast<size_t>(b) * (nx + 1);
      for (int x = 0; x < nx; ++x)
        pref[static_cast<size_t>(p + 1) * nx + x] =
            pref[static_cast<size_t>(p) * nx + x] + static_cast<int>(st[x + 1] - st[x]);
    }
    if (q.size() != static_cast<size_t>(2 * s.colour_start[nb]))
      throw DevError(TLSPH_ERR_INTERNAL, "blocked sweep schedule does not cover every cell task twice");
    s.flow_queue.alloc(q.size());
    s.flow_pref.alloc(pref.size());
    s.flow_done.alloc(static_cast<size_t>(nx));
    s.flow_head.alloc(1);
    CK(cudaMemcpyAsync(s.flow_queue.p, q.data(), q.size() * sizeof(int2), cudaMemcpyHostToDevice, s.stream));
    CK(cudaMemcpyAsync(s.flow_pref.p, pref.data(), pref.size() * sizeof(int), cudaMemcpyHostToDevice, s.stream));
    s.sync();
    s.flow_w = w;
    s.flow_k = k;
    s.flow_ntask = static_cast<long long>(q.size());
  }
  Flow fl{};
  fl.queue = s.flow_queue.p;
  fl.ntask = s.flow_ntask;
  fl.pref = s.flow_pref.p;
  fl.done = s.flow_done.p;
  fl.head = s.flow_head.p;
  fl.nb = nb;
  return fl;
}

template <int D>
void enqueue_sweep_blocked(DevSystem& s, int scheme, const Phase& ph, int w, int k) {
  const int K = (s.max_row + kWarp - 1) / kWarp;
  if (scheme == TLSPH_SCHEME_PARTICLE_SPLIT && s.reduction != TLSPH_REDUCTION_ORDERED && K <= 4) {
    const Flow fl = flow_schedule<D>(s, w, k);
    CK(cudaMemsetAsync(s.flow_done.p, 0, static_cast<size_t>(s.dims[0]) * sizeof(int), s.stream));
    CK(cudaMemsetAsync(s.flow_head.p, 0, sizeof(unsigned long long), s.stream));
    const DFields f = s.fields();
    Phase pf = ph;
    pf.ncol = pf.ncol_colour = s.colour_start[1] - s.colour_start[0];  // the staged/streamed choice
    for (int b = 1; b < colour_count<D>(); ++b)
      pf.ncol_colour = std::max(pf.ncol_colour, s.colour_start[b + 1] - s.colour_start[b]);
    pf.ncol = pf.ncol_colour;
    if (K <= 1) launch_flow<D, 1>(s, f, pf, fl);
    else if (K == 2) launch_flow<D, 2>(s, f, pf, fl);
    else if (K == 3) launch_flow<D, 3>(s, f, pf, fl);
    else launch_flow<D, 4>(s, f, pf, fl);
    return;
  }
  // other schemes and modes: the same order as a sequence of column-range launches
  blocked_order<D>(s.dims[0], w, k,
                   [&](int p, int xa, int xb) { enqueue_phase_columns<D>(s, scheme, ph, p, xa, xb); });
}

template <int D>
void enqueue_sweep_d(DevSystem& s, int scheme, double eta, double dt, bool from_scal) {
  const Phase ph = prepare_sweep<D>(s, scheme, eta, dt, from_scal);
  const auto [w, k] = sweep_blocking<D>(s, scheme);
  if (w > 0) {
    enqueue_sweep_blocked<D>(s, scheme, ph, w, k);
  } else {
    for (int pass = 0; pass < 2; ++pass)
      for (int bb = 0; bb < colour_count<D>(); ++bb) enqueue_phase<D>(s, scheme, ph, pass, bb);
  }
  CK_LAUNCH("k_sweep_phase");
}

// ------------------------------------------------------------------ x-slab halo columns
// Particles of cell column x in (z, y, cell order): the same sequence on every
// rank that holds the column (cells keep ascending reference ids).
// Component c of particle p of a column field lives at ptr[c][p * stride[c]].
struct ColumnField {
  double* ptr[10];
  int ncomp;
  long long stride[10];
};

__global__ void k_column_copy(const long long* __restrict__ cell_start, const long long* __restrict__ col_off,
                              int x, int dims0, int ncol_cells, ColumnField cf, double* __restrict__ buf,
                              long long count, int pack) {
  const int q = blockIdx.x;  // (y, z) cell of the column
  if (q >= ncol_cells) return;
  const long long lin = static_cast<long long>(q) * dims0 + x;
  const long long p0 = cell_start[lin], p1 = cell_start[lin + 1];
  const long long o = col_off[q];
  for (long long e = threadIdx.x; e < p1 - p0; e += blockDim.x)
    for (int c = 0; c < cf.ncomp; ++c) {
      double* a = cf.ptr[c] + (p0 + e) * cf.stride[c];
      if (pack) buf[c * count + o + e] = *a;
      else *a = buf[c * count + o + e];
    }
}

// Bit-for-bit check of div_by against IEEE division on the device.
__global__ void k_selftest_division(unsigned long long seed, long long n, unsigned long long* bad) {
  unsigned long long s = seed ^ (0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1));
  auto next = [&]() {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    return s;
  };
  unsigned long long local = 0;
  for (long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const unsigned long long ea = 1023 - 40 + next() % 81, eb = 1023 - 40 + next() % 81;
    unsigned long long ma = next(), mb = next();
    if (next() & 1) ma &= 0xFFFF;
    if (next() & 1) mb |= 0xFFFFFFFFFFFF0ull;
    const double a = __longlong_as_double(static_cast<long long>((ea << 52) | (ma & 0xFFFFFFFFFFFFFull) |
                                                                 ((next() & 1) << 63)));
    const double b = __longlong_as_double(static_cast<long long>((eb << 52) | (mb & 0xFFFFFFFFFFFFFull)));
    const double y = 1.0 / b;
    if (div_by(a, b, y) != a / b) ++local;
  }
  if (local) atomicAdd(bad, local);
}

}  // namespace

void DevSystem::prepare_sweep_schedule(int scheme) {
  auto build = [&](auto dim) {
    constexpr int DD = decltype(dim)::value;
    const auto [w, k] = sweep_blocking<DD>(*this, scheme);
    const int K = (max_row + kWarp - 1) / kWarp;
    if (w > 0 && scheme == TLSPH_SCHEME_PARTICLE_SPLIT && reduction != TLSPH_REDUCTION_ORDERED && K <= 4)
      flow_schedule<DD>(*this, w, k);
  };
  if (D == 2) build(std::integral_constant<int, 2>{});
  else build(std::integral_constant<int, 3>{});
}

void DevSystem::enqueue_sweep(int scheme, double eta_tilde, double dt_fixed, bool dt_from_scalars) {
  if (D == 2) enqueue_sweep_d<2>(*this, scheme, eta_tilde, dt_fixed, dt_from_scalars);
  else enqueue_sweep_d<3>(*this, scheme, eta_tilde, dt_fixed, dt_from_scalars);
}

// Peer indices for the columns this slab shares with `peer` on `side` (0: left,
// 1: right): both hold the columns' particles, binned in the same global cells
// with the same in-cell order, so the k-th particle of a cell maps to the k-th.
void DevSystem::link_peer(int side, DevSystem& peer) {
  if (!peer.grid_given || peer.D != D || peer.ncells != ncells)
    throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "peers must be slabs of the same global grid");
  double* pv[3] = {nullptr, nullptr, nullptr};
  for (int d = 0; d < D; ++d) pv[d] = peer.v[d].p;
  link_peer_arrays(side, peer.cell_start_h.data(), pv);
}

// The peer given by its cell table (host, ncells + 1 entries) and velocity arrays (device
// pointers reachable from this slab's GPU: the peer's own, or opened from its IPC export).
void DevSystem::link_peer_arrays(int side, const long long* peer_cell_start, double* const* peer_vel) {
  if (side != 0 && side != 1) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "peer side must be 0 (left) or 1 (right)");
  if (!grid_given) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "peers must be slabs of the same global grid");
  const int x0 = task_x0, x1 = task_x1 < 0 ? dims[0] : task_x1;
  // shared columns: left x0-1 (peer owns) and x0 (we own); right x1-1 (we own) and x1 (peer owns)
  const int ca = side == 0 ? x0 - 1 : x1 - 1, cb = ca + 1;
  if (ca < 0 || cb >= dims[0]) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "no neighbouring slab on that side");
  std::vector<int> idx(static_cast<size_t>(n), -1);
  if (peer_idx.p) CK(cudaMemcpy(idx.data(), peer_idx.p, idx.size() * sizeof(int), cudaMemcpyDeviceToHost));
  const int nq = static_cast<int>(ncells / dims[0]);
  for (int x : {ca, cb})
    for (int q = 0; q < nq; ++q) {
      const long long lin = static_cast<long long>(q) * dims[0] + x;
      const long long a0 = cell_start_h[lin], a1 = cell_start_h[lin + 1];
      const long long b0 = peer_cell_start[lin], b1 = peer_cell_start[lin + 1];
      if (a1 - a0 != b1 - b0) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "peer slabs disagree on a shared cell");
      for (long long k = 0; k < a1 - a0; ++k) {
        const long long j = b0 + k;
        idx[static_cast<size_t>(a0 + k)] = side == 1 ? static_cast<int>(j) : -2 - static_cast<int>(j);
      }
    }
  peer_idx.alloc(idx.size());
  CK(cudaMemcpy(peer_idx.p, idx.data(), idx.size() * sizeof(int), cudaMemcpyHostToDevice));
  for (int d = 0; d < 3; ++d) peer_v[side][d] = d < D ? peer_vel[d] : nullptr;
  peer_x[side] = side == 0 ? x0 : x1 - 1;
}

// ---- cross-process linking (one process per GPU)
void DevSystem::ensure_phase_events(bool interprocess) {
  const int nphase = 2 * (D == 2 ? 9 : 27);
  if (interprocess && !phase_events_ipc) {
    for (cudaEvent_t e : phase_events) cudaEventDestroy(e);
    phase_events.clear();
  }
  CK(cudaSetDevice(device));
  while (static_cast<int>(phase_events.size()) < nphase) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | (interprocess ? cudaEventInterprocess : 0)));
    phase_events.push_back(e);
  }
  if (interprocess) {
    phase_events_ipc = true;
    for (cudaEvent_t& e : halo_events)
      if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventInterprocess));
  }
}

void DevSystem::ipc_export(IpcExport* out) {
  ensure_phase_events(true);
  std::memset(out, 0, sizeof(IpcExport));
  out->magic = IpcExport::kMagic;
  out->dim = D;
  out->device = device;
  out->nphase = static_cast<int>(phase_events.size());
  out->n = n;
  for (int d = 0; d < D; ++d) CK(cudaIpcGetMemHandle(&out->vel[d], v[d].p));
  CK(cudaIpcGetMemHandle(&out->pbv, pbv.p));
  for (int q = 0; q < out->nphase; ++q) CK(cudaIpcGetEventHandle(&out->ev[q], phase_events[q]));
  for (int k = 0; k < 3; ++k) CK(cudaIpcGetEventHandle(&out->hev[k], halo_events[k]));
}

void DevSystem::link_peer_ipc(int side, const IpcExport& peer, const long long* peer_cell_start) {
  if (peer.magic != IpcExport::kMagic || peer.dim != D)
    throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "not an IPC export of a slab of this dimension");
  if (side != 0 && side != 1) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "peer side must be 0 (left) or 1 (right)");
  CK(cudaSetDevice(device));
  IpcPeer& ip = ipc_peer[side];
  ip.close();
  double* pv[3] = {nullptr, nullptr, nullptr};
  for (int d = 0; d < D; ++d) {
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, peer.vel[d], cudaIpcMemLazyEnablePeerAccess));
    ip.mem.push_back(p);
    pv[d] = static_cast<double*>(p);
  }
  for (int q = 0; q < peer.nphase; ++q) {
    cudaEvent_t e;
    CK(cudaIpcOpenEventHandle(&e, peer.ev[q]));
    ip.ev.push_back(e);
  }
  {
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, peer.pbv, cudaIpcMemLazyEnablePeerAccess));
    ip.mem.push_back(p);
    ip.pbv = static_cast<double*>(p);
    ip.n = peer.n;
  }
  for (int k = 0; k < 3; ++k) CK(cudaIpcOpenEventHandle(&ip.hev[k], peer.hev[k]));
  link_peer_arrays(side, peer_cell_start, pv);
}

void IpcPeer::close() {
  for (void* p : mem) cudaIpcCloseMemHandle(p);
  for (cudaEvent_t e : ev) cudaEventDestroy(e);
  for (cudaEvent_t& e : hev)
    if (e) {
      cudaEventDestroy(e);
      e = nullptr;
    }
  mem.clear();
  ev.clear();
  pbv = nullptr;
}

// Phase q of the decomposed sweep of this slab, asynchronous: the stream first waits on the
// linked neighbours' events of phase `wait_q` (-1: none), then runs the phase and records
// its own event q. The caller orders the calls so a neighbour recorded wait_q before.
void DevSystem::sweep_phase_ipc(int scheme, double eta_tilde, double dt, int q, int wait_q) {
  ensure_phase_events(true);
  const int nphase = static_cast<int>(phase_events.size());
  if (q < 0 || q >= nphase || wait_q >= nphase) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "phase out of range");
  CK(cudaSetDevice(device));
  if (wait_q >= 0)
    for (int side = 0; side < 2; ++side)
      if (!ipc_peer[side].ev.empty()) CK(cudaStreamWaitEvent(stream, ipc_peer[side].ev[wait_q], 0));
  if (eta_tilde != 0.0) enqueue_sweep_phase(scheme, eta_tilde, dt, q < nphase / 2 ? 0 : 1, q % (nphase / 2));
  CK(cudaEventRecord(phase_events[q], stream));
}

void DevSystem::build_colour_lists() {
  std::vector<long long> cst(static_cast<size_t>(ncells + 1));
  CK(cudaMemcpyAsync(cst.data(), cell_start.p, cst.size() * sizeof(long long), cudaMemcpyDeviceToHost, stream));
  sync();
  const int x0 = task_x0, x1 = task_x1 < 0 ? dims[0] : std::min(task_x1, dims[0]);
  const int nb = D == 2 ? 9 : 27;
  const int nx = dims[0];
  std::vector<int> cells, xcells;
  colour_start.assign(static_cast<size_t>(nb + 1), 0);
  xcol_start.assign(static_cast<size_t>(nb) * (nx + 1), 0);
  std::vector<std::pair<long long, int>> col;  // (-count, cell)
  std::vector<std::tuple<int, long long, int>> bycol;  // (x, -count, cell)
  for (int b = 0; b < nb; ++b) {
    const int r0 = b % 3, r1 = (b / 3) % 3, r2 = D == 3 ? b / 9 : 0;
    col.clear();
    bycol.clear();
    for (int z = r2; z < (D == 3 ? dims[2] : 1); z += 3)
      for (int y = r1; y < dims[1]; y += 3)
        for (int x = r0; x < dims[0]; x += 3) {
          if (x < x0 || x >= x1) continue;
          const long long lin = (static_cast<long long>(z) * dims[1] + y) * dims[0] + x;
          const long long cnt = cst[lin + 1] - cst[lin];
          if (cnt > 0) {
            col.emplace_back(-cnt, static_cast<int>(lin));
            bycol.emplace_back(x, -cnt, static_cast<int>(lin));
          }
        }
    std::stable_sort(col.begin(), col.end());
    colour_start[b] = static_cast<long long>(cells.size());
    for (const auto& c : col) cells.push_back(c.second);
    std::stable_sort(bycol.begin(), bycol.end());
    long long* xs = xcol_start.data() + static_cast<size_t>(b) * (nx + 1);
    size_t k = 0;
    for (int x = 0; x <= nx; ++x) {
      while (k < bycol.size() && std::get<0>(bycol[k]) < x) xcells.push_back(std::get<2>(bycol[k++]));
      xs[x] = static_cast<long long>(xcells.size());
    }
  }
  colour_start[nb] = static_cast<long long>(cells.size());
  colour_cells.alloc(std::max<size_t>(cells.size(), 1));
  xcol_cells.alloc(std::max<size_t>(xcells.size(), 1));
  xcol_cells_h = xcells;
  flow_ntask = 0;  // the dataflow schedule is rebuilt from the new lists
  if (!cells.empty()) {
    CK(cudaMemcpyAsync(colour_cells.p, cells.data(), cells.size() * sizeof(int), cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(xcol_cells.p, xcells.data(), xcells.size() * sizeof(int), cudaMemcpyHostToDevice, stream));
  }
  sync();
}

// Ownership of a slab's particles: those of the task columns [x0, x1). The
// whole grid as task range (or no slab) clears the mask: every particle owned.
void DevSystem::build_own_mask() {
  const int x0 = task_x0, x1 = task_x1 < 0 ? dims[0] : std::min(task_x1, dims[0]);
  if (x0 <= 0 && x1 >= dims[0]) {
    own.release();
    return;
  }
  std::vector<uint8_t> m(static_cast<size_t>(n), 0);
  for (long long lin = 0; lin < ncells; ++lin) {
    const int x = static_cast<int>(lin % dims[0]);
    if (x < x0 || x >= x1) continue;
    for (long long p = cell_start_h[lin]; p < cell_start_h[lin + 1]; ++p) m[static_cast<size_t>(p)] = 1;
  }
  own.alloc(m.size());
  CK(cudaMemcpy(own.p, m.data(), m.size(), cudaMemcpyHostToDevice));
}

void DevSystem::enqueue_sweep_phase(int scheme, double eta_tilde, double dt_fixed, int pass, int index) {
  const int nb = D == 2 ? 9 : 27;
  if (pass < 0 || pass > 1 || index < 0 || index >= nb)
    throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "colour phase out of range");
  if (D == 2) enqueue_phase<2>(*this, scheme, prepare_sweep<2>(*this, scheme, eta_tilde, dt_fixed, false), pass, index);
  else enqueue_phase<3>(*this, scheme, prepare_sweep<3>(*this, scheme, eta_tilde, dt_fixed, false), pass, index);
  CK_LAUNCH("k_sweep_phase");
}

// Sweeps over peer-linked slabs with the per-phase ordering on the devices (tlsph_dev_sweep_linked).
// Phase q of slab r may start once phase q-1 of slabs r-1 and r+1 has finished: they store into
// r's shared columns (fused exchange) and read the columns r stores into theirs. Events are
// recorded and waited in host program order, so every wait refers to the intended phase.
void sweep_linked(const std::vector<DevSystem*>& sl, int scheme, double eta_tilde, double dt, int count) {
  if (sl.empty()) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "no slabs");
  const int D0 = sl[0]->D;
  for (DevSystem* s : sl)
    if (!s || s->D != D0) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "slabs must share the dimension");
  const int nphase = 2 * (D0 == 2 ? 9 : 27);
  for (DevSystem* s : sl) {
    CK(cudaSetDevice(s->device));
    while (static_cast<int>(s->phase_events.size()) < nphase) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      s->phase_events.push_back(e);
    }
  }
  DevSystem& s0 = *sl[0];
  CK(cudaSetDevice(s0.device));
  cudaEvent_t t0, t1;
  CK(cudaEventCreate(&t0));
  CK(cudaEventCreate(&t1));
  CK(cudaEventRecord(t0, s0.stream));
  for (size_t r = 1; r < sl.size(); ++r) {  // every slab starts after t0
    CK(cudaSetDevice(sl[r]->device));
    CK(cudaStreamWaitEvent(sl[r]->stream, t0, 0));
  }
  const int nr = static_cast<int>(sl.size());
  for (int c = 0; c < count; ++c) {
    for (int q = 0; q < nphase; ++q) {
      const int pass = q < nphase / 2 ? 0 : 1, index = q % (nphase / 2);
      for (int r = 0; r < nr; ++r) {
        DevSystem& s = *sl[r];
        CK(cudaSetDevice(s.device));
        const bool first = c == 0 && q == 0;
        if (!first) {
          const int qp = q > 0 ? q - 1 : nphase - 1;  // the previous phase (of the previous sweep)
          if (r > 0) CK(cudaStreamWaitEvent(s.stream, sl[r - 1]->phase_events[qp], 0));
          if (r + 1 < nr) CK(cudaStreamWaitEvent(s.stream, sl[r + 1]->phase_events[qp], 0));
        }
        s.enqueue_sweep_phase(scheme, eta_tilde, dt, pass, index);
        CK(cudaEventRecord(s.phase_events[q], s.stream));
      }
    }
  }
  CK(cudaSetDevice(s0.device));
  for (int r = 1; r < nr; ++r) CK(cudaStreamWaitEvent(s0.stream, sl[r]->phase_events[nphase - 1], 0));
  CK(cudaEventRecord(t1, s0.stream));
  CK(cudaEventSynchronize(t1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, t0, t1));
  s0.last_elapsed = ms * 1e-3;
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  for (DevSystem* s : sl) {
    CK(cudaSetDevice(s->device));
    CK(cudaStreamSynchronize(s->stream));
  }
  CK(cudaSetDevice(s0.device));
}

namespace {
// cell count of a column and the exclusive prefix of its cells' particle counts
std::vector<long long> column_offsets(const DevSystem& s, int x) {
  if (!s.grid_given) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "column transfer needs a slab system (given grid)");
  if (x < 0 || x >= s.dims[0]) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "column out of range");
  const int nq = static_cast<int>(s.ncells / s.dims[0]);
  std::vector<long long> off(static_cast<size_t>(nq) + 1, 0);
  for (int q = 0; q < nq; ++q) {
    const long long lin = static_cast<long long>(q) * s.dims[0] + x;
    off[q + 1] = off[q] + (s.cell_start_h[lin + 1] - s.cell_start_h[lin]);
  }
  return off;
}

ColumnField column_field(const DevSystem& s, int field) {
  ColumnField cf{};
  if (field == TLSPH_DEV_COLUMN_VELOCITY) {
    cf.ncomp = s.D;
    for (int d = 0; d < s.D; ++d) {
      cf.ptr[d] = s.v[d].p;
      cf.stride[d] = 1;
    }
  } else if (field == TLSPH_DEV_COLUMN_STRESS) {
    cf.ncomp = s.D * s.D + 1;  // P B0 row-major, V0 (the packed momentum-gather record)
    // component c of particle p at pbv_at(n, p, c) = ptr[c] + p * stride[c]
    const auto at = [&](long long p, int c) { return s.D == 2 ? pbv_at<2>(s.n, p, c) : pbv_at<3>(s.n, p, c); };
    for (int c = 0; c < cf.ncomp; ++c) {
      cf.ptr[c] = s.pbv.p + at(0, c);
      cf.stride[c] = at(1, c) - at(0, c);
    }
  } else {
    throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "unknown column field " + std::to_string(field));
  }
  return cf;
}

void column_copy(DevSystem& s, int field, int x, double* buf, bool pack) {
  const ColumnField cf = column_field(s, field);
  const std::vector<long long> off = column_offsets(s, x);
  const int nq = static_cast<int>(off.size()) - 1;
  const long long count = off.back();
  if (count == 0) return;
  DBuf<long long> doff;
  doff.alloc(off.size());
  CK(cudaMemcpyAsync(doff.p, off.data(), off.size() * sizeof(long long), cudaMemcpyHostToDevice, s.stream));
  k_column_copy<<<static_cast<unsigned>(nq), 64, 0, s.stream>>>(s.cell_start.p, doff.p, x, s.dims[0], nq, cf, buf,
                                                                count, pack ? 1 : 0);
  CK_LAUNCH("k_column_copy");
  s.sync();  // the buffer is handed to another stream / library (NCCL, torch)
}
}  // namespace

long long DevSystem::column_count(int x) const { return column_offsets(*this, x).back(); }
// Halo push of a cross-process slab (tlsph_dev_push_halo_ipc): the particles of our owned boundary
// column x, stored straight into the neighbour's copy of that column (its halo) through the IPC
// mapping, at the indices link_peer_arrays recorded (peer_idx: >= 0 right peer, <= -2 left).
__global__ void k_column_push(const long long* __restrict__ cell_start, int x, int dims0, int ncol_cells,
                              ColumnField src, ColumnField dst, const int* __restrict__ peer_idx) {
  const int q = blockIdx.x;
  if (q >= ncol_cells) return;
  const long long lin = static_cast<long long>(q) * dims0 + x;
  for (long long p = cell_start[lin] + threadIdx.x; p < cell_start[lin + 1]; p += blockDim.x) {
    const int pi = peer_idx[p];
    if (pi == -1) continue;
    const long long idx = pi >= 0 ? pi : -2 - pi;
    for (int c = 0; c < src.ncomp; ++c) dst.ptr[c][idx * dst.stride[c]] = src.ptr[c][p * src.stride[c]];
  }
}

// The neighbour's side of a column field, from its IPC mapping (same layout rules as column_field).
ColumnField peer_column_field(const DevSystem& s, int side, int field) {
  ColumnField cf{};
  const IpcPeer& ip = s.ipc_peer[side];
  if (field == TLSPH_DEV_COLUMN_VELOCITY) {
    cf.ncomp = s.D;
    for (int d = 0; d < s.D; ++d) {
      cf.ptr[d] = s.peer_v[side][d];
      cf.stride[d] = 1;
    }
  } else {
    cf.ncomp = s.D * s.D + 1;
    const auto at = [&](long long p, int c) { return s.D == 2 ? pbv_at<2>(ip.n, p, c) : pbv_at<3>(ip.n, p, c); };
    for (int c = 0; c < cf.ncomp; ++c) {
      cf.ptr[c] = ip.pbv + at(0, c);
      cf.stride[c] = at(1, c) - at(0, c);
    }
  }
  return cf;
}

void DevSystem::push_halo_ipc(int field) {
  if (field != TLSPH_DEV_COLUMN_VELOCITY && field != TLSPH_DEV_COLUMN_STRESS)
    throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "unknown column field " + std::to_string(field));
  ensure_phase_events(true);
  CK(cudaSetDevice(device));
  const int x0 = task_x0, x1 = task_x1 < 0 ? dims[0] : task_x1;
  const int nq = static_cast<int>(ncells / dims[0]);
  const ColumnField src = column_field(*this, field);
  for (int side = 0; side < 2; ++side) {
    if (ipc_peer[side].ev.empty()) continue;
    const ColumnField dst = peer_column_field(*this, side, field);
    if (dst.ncomp != src.ncomp) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "peer column layout differs");
    k_column_push<<<static_cast<unsigned>(nq), 64, 0, stream>>>(cell_start.p, side == 0 ? x0 : x1 - 1, dims[0], nq,
                                                               src, dst, peer_idx.p);
  }
  CK_LAUNCH("k_column_push");
  CK(cudaEventRecord(halo_events[field], stream));
}

void DevSystem::wait_halo_ipc(int field) {
  if (field != TLSPH_DEV_COLUMN_VELOCITY && field != TLSPH_DEV_COLUMN_STRESS)
    throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "unknown column field " + std::to_string(field));
  CK(cudaSetDevice(device));
  for (int side = 0; side < 2; ++side)
    if (ipc_peer[side].hev[field]) CK(cudaStreamWaitEvent(stream, ipc_peer[side].hev[field], 0));
}

// Cross-process ordering points that carry no data. mark_ipc records this slab's mark event after
// everything enqueued so far (e.g. verlet pass C, which reads the velocities the neighbours' first
// sweep phase stores into); wait_mark_ipc puts the neighbours' marks in front of this slab's next
// work. wait_phase_ipc(q) makes the stream wait on the neighbours' phase-q events, so a sweep ends
// only after every store of theirs into this slab landed. Host ordering as for the halo pushes.
void DevSystem::mark_ipc() {
  ensure_phase_events(true);
  CK(cudaSetDevice(device));
  CK(cudaEventRecord(halo_events[2], stream));
}

void DevSystem::wait_mark_ipc() {
  CK(cudaSetDevice(device));
  for (int side = 0; side < 2; ++side)
    if (ipc_peer[side].hev[2]) CK(cudaStreamWaitEvent(stream, ipc_peer[side].hev[2], 0));
}

void DevSystem::wait_phase_ipc(int q) {
  CK(cudaSetDevice(device));
  for (int side = 0; side < 2; ++side) {
    const IpcPeer& ip = ipc_peer[side];
    if (ip.ev.empty()) continue;
    if (q < 0 || q >= static_cast<int>(ip.ev.size())) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "phase out of range");
    CK(cudaStreamWaitEvent(stream, ip.ev[q], 0));
  }
}

int DevSystem::column_width(int field) const { return column_field(*this, field).ncomp; }
void DevSystem::pack_column(int field, int x, double* dev_dst) { column_copy(*this, field, x, dev_dst, true); }
void DevSystem::unpack_column(int field, int x, const double* dev_src) {
  column_copy(*this, field, x, const_cast<double*>(dev_src), false);
}

unsigned long long selftest_division(long long n, unsigned long long seed) {
  DBuf<unsigned long long> bad;
  bad.alloc(1);
  CK(cudaMemset(bad.p, 0, sizeof(unsigned long long)));
  k_selftest_division<<<592, 256>>>(seed, n, bad.p);
  CK_LAUNCH("k_selftest_division");
  unsigned long long h = 0;
  CK(cudaMemcpy(&h, bad.p, sizeof(h), cudaMemcpyDeviceToHost));
  return h;
}

}  // namespace tlsph_cuda

#ifdef TLSPH_SWEEP_TIMING
extern "C" int tlsph_debug_sweep_stamps(unsigned long long* out, int cells) {
  const int n = cells < (1 << 16) ? cells : (1 << 16);
  return cudaMemcpyFromSymbol(out, tlsph_cuda::g_sweep_stamp,
                              sizeof(unsigned long long) * tlsph_cuda::kStampSlots * n) == cudaSuccess
             ? n
             : -1;
}
#endif
