#include <atomic>
// Device system construction: the GPU splitting cell-linked list.
//
//   bbox -> cell keys -> counting sort (histogram, exclusive scan, scatter,
//   per-cell id sort = stable order) -> sorted SoA gather -> reference-
//   configuration CSR (count, scan, warp-per-particle fill with ascending
//   reference-j order and bit-exact pair geometry).
//
// Reference: proj/src/tlsph/neighbors.cpp:14-141 (build_cell_grid,
// block_decompose, build_reference_neighborhoods), particle_system.hpp:32-45.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "hostio.cuh"
#include "system.cuh"

namespace tlsph_cuda {

// Bytes moved between the caller's host memory and the device by field transfers (all handles).
std::atomic<unsigned long long> g_h2d_bytes{0}, g_d2h_bytes{0};


namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr long long kScanTile = kScanThreads * kScanItems;

// ------------------------------------------------------------------ scan
template <typename T>
__global__ void k_scan_tile(const T* __restrict__ in, long long n_in, long long* __restrict__ out, long long n_out,
                            long long* __restrict__ tile_sums) {
  __shared__ long long sh[kScanThreads];
  const long long base = static_cast<long long>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
  long long vals[kScanItems];
  long long local = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const long long idx = base + k;
    const long long x = idx < n_in ? static_cast<long long>(in[idx]) : 0;
    vals[k] = local;
    local += x;
  }
  sh[threadIdx.x] = local;
  __syncthreads();
  for (int off = 1; off < kScanThreads; off <<= 1) {
    const long long add = threadIdx.x >= off ? sh[threadIdx.x - off] : 0;
    __syncthreads();
    sh[threadIdx.x] += add;
    __syncthreads();
  }
  const long long excl = sh[threadIdx.x] - local;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const long long idx = base + k;
    if (idx < n_out) out[idx] = excl + vals[k];
  }
  if (threadIdx.x == kScanThreads - 1) tile_sums[blockIdx.x] = sh[threadIdx.x];
}

__global__ void k_scan_add(long long* out, long long n_out, const long long* tile_offsets) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx < n_out) out[idx] += tile_offsets[idx / kScanTile];
}

// out[0..n] = exclusive scan of in[0..n-1]; out[n] = total.
template <typename T>
void exclusive_scan(const T* in, long long n, long long* out, cudaStream_t st) {
  const long long n_out = n + 1;
  const long long tiles = (n_out + kScanTile - 1) / kScanTile;
  DBuf<long long> sums, sums_scan;
  sums.alloc(static_cast<size_t>(tiles));
  k_scan_tile<T><<<static_cast<unsigned>(tiles), kScanThreads, 0, st>>>(in, n, out, n_out, sums.p);
  CK_LAUNCH("k_scan_tile");
  if (tiles > 1) {
    sums_scan.alloc(static_cast<size_t>(tiles + 1));
    exclusive_scan<long long>(sums.p, tiles, sums_scan.p, st);
    k_scan_add<<<static_cast<unsigned>((n_out + 255) / 256), 256, 0, st>>>(out, n_out, sums_scan.p);
    CK_LAUNCH("k_scan_add");
  }
  CK(cudaStreamSynchronize(st));  // temporaries die here
}

// ------------------------------------------------------------------ cell build
template <int D>
__global__ void k_bbox(const double* __restrict__ r0aos, long long n, double* __restrict__ part, int* bad) {
  __shared__ double smin[D][256], smax[D][256];
  double lo[D], hi[D];
#pragma unroll
  for (int d = 0; d < D; ++d) { lo[d] = INFINITY; hi[d] = -INFINITY; }
  bool nonfinite = false;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const double x = r0aos[i * D + d];
      if (!isfinite(x)) nonfinite = true;
      lo[d] = fmin(lo[d], x);
      hi[d] = fmax(hi[d], x);
    }
  }
  if (nonfinite) atomicOr(bad, 1);
#pragma unroll
  for (int d = 0; d < D; ++d) { smin[d][threadIdx.x] = lo[d]; smax[d][threadIdx.x] = hi[d]; }
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (threadIdx.x < off)
#pragma unroll
      for (int d = 0; d < D; ++d) {
        smin[d][threadIdx.x] = fmin(smin[d][threadIdx.x], smin[d][threadIdx.x + off]);
        smax[d][threadIdx.x] = fmax(smax[d][threadIdx.x], smax[d][threadIdx.x + off]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
#pragma unroll
    for (int d = 0; d < D; ++d) {
      part[blockIdx.x * 2 * D + d] = smin[d][0];
      part[blockIdx.x * 2 * D + D + d] = smax[d][0];
    }
}

template <int D>
__global__ void k_cell_keys(const double* __restrict__ r0aos, long long n, DFields f, int* __restrict__ key,
                            int* __restrict__ count) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[D];
#pragma unroll
  for (int d = 0; d < D; ++d) p[d] = r0aos[i * D + d];
  int c[D];
  cell_coords<D>(p, f.origin, f.cell, f.dims, c);
  const int k = static_cast<int>(cell_linear<D>(c, f.dims));
  key[i] = k;
  atomicAdd(&count[k], 1);
}

__global__ void k_cell_scatter(const int* __restrict__ key, long long n, const long long* __restrict__ cell_start,
                               int* __restrict__ fill, int* __restrict__ perm) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int k = key[i];
  const long long pos = cell_start[k] + atomicAdd(&fill[k], 1);
  perm[pos] = static_cast<int>(i);
}

// Current-position cell key of every particle (the per-step re-sort, DevSystem::enqueue_resort).
template <int D>
__global__ void k_cell_keys_current(DFields f, int* __restrict__ key, int* __restrict__ count) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= f.n) return;
  double p[D];
#pragma unroll
  for (int d = 0; d < D; ++d) p[d] = f.r[d][i];
  int c[D];
  cell_coords<D>(p, f.origin, f.cell, f.dims, c);
  const int k = static_cast<int>(cell_linear<D>(c, f.dims));
  key[i] = k;
  atomicAdd(&count[k], 1);
}

// Insertion sort of each cell's ids: the atomic scatter above is unordered,
// the reference lists ascending ids per cell (neighbors.cpp:52-57).
__global__ void k_cell_sort(const long long* __restrict__ cell_start, long long ncells, int* __restrict__ perm,
                            int* __restrict__ max_cell) {
  const long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  const long long s = cell_start[c], e = cell_start[c + 1];
  for (long long a = s + 1; a < e; ++a) {
    const int x = perm[a];
    long long b = a - 1;
    while (b >= s && perm[b] > x) {
      perm[b + 1] = perm[b];
      --b;
    }
    perm[b + 1] = x;
  }
  atomicMax(max_cell, static_cast<int>(e - s));
}

template <int D>
__global__ void k_gather_init(DFields f, const double* __restrict__ r0aos, const double* __restrict__ V0h,
                              const double* __restrict__ rho0h, const uint8_t* __restrict__ cons) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= f.n) return;
  const int i = f.perm[s];
  f.rank[i] = static_cast<int>(s);
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double x = r0aos[static_cast<long long>(i) * D + d];
    f.r0[d][s] = x;
    f.r[d][s] = x;
    f.v[d][s] = 0.0;
    f.a[d][s] = 0.0;
    f.body[d][s] = 0.0;
  }
#pragma unroll
  for (int k = 0; k < D * D; ++k) {
    const double id = (k % (D + 1) == 0) ? 1.0 : 0.0;
    f.F[k][s] = id;
    f.dFdt[k][s] = 0.0;
    f.B0[k][s] = id;
  }
  const double vol = V0h[i], dens = rho0h[i];
#pragma unroll
  for (int k = 0; k < pbv_stride<D>(); ++k) f.pbv[pbv_at<D>(f.n, s, k)] = 0.0;
  f.pbv[pbv_at<D>(f.n, s, D * D)] = vol;
  f.V0[s] = vol;
  f.m[s] = dens * vol;  // particle_system.hpp:40
  f.rho0[s] = dens;
  f.rho[s] = dens;
  f.flag[s] = cons ? cons[i] : 0;
  const double r = 1.0 / f.m[s];
  f.minvf[s] = f.flag[s] ? -r : r;
}

// ------------------------------------------------------------------ neighbourhoods
template <int D>
__device__ __forceinline__ double pair_dist(const DFields& f, long long i, long long j, double* diff) {
#pragma unroll
  for (int d = 0; d < D; ++d) diff[d] = f.r0[d][i] - f.r0[d][j];
  double s = diff[0] * diff[0];
#pragma unroll
  for (int d = 1; d < D; ++d) s = s + diff[d] * diff[d];
  return sqrt(s);
}

template <int D>
__device__ __forceinline__ void stencil_cell(const int* base, int s, const int* dims, int* c, bool& ok) {
  int rem = s;
  ok = true;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    c[d] = base[d] + (rem % 3) - 1;
    rem /= 3;
    if (c[d] < 0 || c[d] >= dims[d]) ok = false;
  }
}

// Per particle: accepted-neighbour count (dist < cutoff, neighbors.cpp:92-115),
// staged-stencil size, coincident-pair detection.
template <int D>
__global__ void k_nbr_count(DFields f, double cutoff, int* __restrict__ counts, int* __restrict__ max_stencil,
                            DScalars* sc) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= f.n) return;
  double p[D];
#pragma unroll
  for (int d = 0; d < D; ++d) p[d] = f.r0[d][i];
  int base[D];
  cell_coords<D>(p, f.origin, f.cell, f.dims, base);
  int cnt = 0;
  constexpr int kStencil = D == 2 ? 9 : 27;
  for (int s = 0; s < kStencil; ++s) {
    int c[D];
    bool ok;
    stencil_cell<D>(base, s, f.dims, c, ok);
    if (!ok) continue;
    const long long lin = cell_linear<D>(c, f.dims);
    const long long b = f.cell_start[lin], e = f.cell_start[lin + 1];
    for (long long j = b; j < e; ++j) {
      if (j == i) continue;
      double diff[D];
      const double dist = pair_dist<D>(f, i, j, diff);
      if (dist >= cutoff) continue;
      if (!(dist > 0.0)) {
        const unsigned long long key = (static_cast<unsigned long long>(f.perm[i]) << 32) |
                                       (static_cast<unsigned long long>(s) << 24) |
                                       static_cast<unsigned long long>(j - b);
        record_error(sc, ERR_COINCIDENT, key);
      }
      ++cnt;
    }
  }
  counts[i] = cnt;
  Stencil<D> st;
  stencil_segments<D>(f.cell_start, f.dims, base, st);
  atomicMax(max_stencil, st.total);
}

// Warp per particle: gather accepted candidates in stencil-scan order, rank
// them by reference id (the reference std::sort, neighbors.cpp:116), write
// the slot geometry with the reference's arithmetic (neighbors.cpp:118-139).
template <int D>
__global__ void k_nbr_fill(DFields f, double cutoff, double h, double sigma, int cap) {
  extern __shared__ unsigned char smem_raw[];
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const int warps = blockDim.x / kWarp;
  int* s_ref = reinterpret_cast<int*>(smem_raw) + warp * cap;
  int* s_idx = reinterpret_cast<int*>(smem_raw) + warps * cap + warp * cap;
  uint16_t* s_loc = reinterpret_cast<uint16_t*>(reinterpret_cast<int*>(smem_raw) + 2 * warps * cap) + warp * cap;
  const long long i = static_cast<long long>(blockIdx.x) * warps + warp;
  if (i >= f.n) return;
  double p[D];
#pragma unroll
  for (int d = 0; d < D; ++d) p[d] = f.r0[d][i];
  int base[D];
  cell_coords<D>(p, f.origin, f.cell, f.dims, base);
  Stencil<D> st;
  stencil_segments<D>(f.cell_start, f.dims, base, st);
  int count = 0;
  constexpr int kStencil = D == 2 ? 9 : 27;
  for (int s = 0; s < kStencil; ++s) {
    int c[D];
    bool ok;
    stencil_cell<D>(base, s, f.dims, c, ok);
    if (!ok) continue;
    const long long lin = cell_linear<D>(c, f.dims);
    const long long b = f.cell_start[lin], e = f.cell_start[lin + 1];
    const int dy = (s / 3) % 3 - 1;
    const int dz = D == 3 ? s / 9 - 1 : 0;
    const int seg = D == 2 ? dy + 1 : (dz + 1) * 3 + (dy + 1);
    for (long long j0 = b; j0 < e; j0 += kWarp) {
      const long long j = j0 + lane;
      bool acc = false;
      if (j < e && j != i) {
        double diff[D];
        acc = pair_dist<D>(f, i, j, diff) < cutoff;
      }
      const unsigned mask = __ballot_sync(0xffffffffu, acc);
      if (acc) {
        const int pos = count + __popc(mask & ((1u << lane) - 1u));
        if (pos < cap) {
          s_ref[pos] = f.perm[j];
          s_idx[pos] = static_cast<int>(j);
          const long long loc = st.base[seg] + (j - st.start[seg]);
          s_loc[pos] = loc < kNoLocal ? static_cast<uint16_t>(loc) : kNoLocal;
        }
      }
      count += __popc(mask);
    }
  }
  __syncwarp();
  const long long row = f.offs[i];
  for (int k = lane; k < count && k < cap; k += kWarp) {
    const int ref = s_ref[k];
    int rank = 0;
    for (int q = 0; q < count; ++q) rank += s_ref[q] < ref ? 1 : 0;
    const long long slot = row + rank;
    const long long j = s_idx[k];
    double diff[D];
    const double dist = pair_dist<D>(f, i, j, diff);
    // SmoothingKernel::grad_mag (kernel.cpp:32-38)
    const double q = dist / h;
    double dw = 0.0;
    if (q < 2.0) {
      const double t = 1.0 - 0.5 * q;
      dw = -5.0 * q * (sigma / h) * t * t * t;
    }
    f.nbr[slot] = static_cast<int>(j);
    f.r0_len[slot] = dist;
#pragma unroll
    for (int d = 0; d < D; ++d) f.e0[d][slot] = diff[d] / dist;
    f.dwdr0[slot] = dw;
    f.pf[slot] = 2.0 * f.V0[i] * f.V0[j] * dw / dist;
    f.nloc[slot] = s_loc[k];
  }
}

// ------------------------------------------------------------------ transfers
// Component arrays of one field, passed by value (no device-side pointer table).
struct FieldPtrs {
  double* p[9];
};

__global__ void k_aos_to_soa(const double* __restrict__ src, int comps, long long n, const int* __restrict__ perm,
                             FieldPtrs dst) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const long long i = perm[s];
  for (int c = 0; c < comps; ++c) dst.p[c][s] = src[i * comps + c];
}

__global__ void k_soa_to_aos(double* __restrict__ dst, int comps, long long n, const int* __restrict__ perm,
                             FieldPtrs src) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const long long i = perm[s];
  for (int c = 0; c < comps; ++c) dst[i * comps + c] = src.p[c][s];
}

// Record transfers in the caller's storage: component c of a D x D matrix (row r = c / D, column
// c % D) sits at c in row-major records and at (c % D) * D + c / D in column-major ones (cm = D).
__device__ __forceinline__ int record_index(int c, int cm) { return cm ? (c % cm) * cm + c / cm : c; }

__global__ void k_records_in(const double* __restrict__ src, int comps, int cm, long long n,
                             const int* __restrict__ perm, FieldPtrs dst) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const long long i = perm[s];
  for (int c = 0; c < comps; ++c) dst.p[c][s] = src[i * comps + record_index(c, cm)];
}

__global__ void k_records_out(double* __restrict__ dst, int comps, int cm, long long n, const int* __restrict__ perm,
                              FieldPtrs src) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const long long i = perm[s];
  for (int c = 0; c < comps; ++c) dst[i * comps + record_index(c, cm)] = src.p[c][s];
}

// Sets *differs when any staged record differs bitwise from the resident field.
__global__ void k_records_differ(const double* __restrict__ src, int comps, int cm, long long n,
                                 const int* __restrict__ perm, FieldPtrs cur, int* differs) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  bool d = false;
  if (s < n) {
    const long long i = perm[s];
    for (int c = 0; c < comps; ++c)
      d = d || __double_as_longlong(src[i * comps + record_index(c, cm)]) != __double_as_longlong(cur.p[c][s]);
  }
  if (__any_sync(0xffffffffu, d) && (threadIdx.x & 31) == 0) atomicOr(differs, 1);
}

__global__ void k_flags_in(const uint8_t* __restrict__ src, long long n, const int* __restrict__ perm, uint8_t* flag,
                           int* differs) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  bool d = false;
  if (s < n) {
    const uint8_t v = src[perm[s]] != 0 ? 1 : 0;
    d = v != flag[s];
    if (!differs) flag[s] = v;
  }
  if (differs && __any_sync(0xffffffffu, d) && (threadIdx.x & 31) == 0) atomicOr(differs, 1);
}

__global__ void k_flags_out(uint8_t* __restrict__ dst, long long n, const int* __restrict__ perm,
                            const uint8_t* __restrict__ flag) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s < n) dst[perm[s]] = flag[s];
}

__global__ void k_minvf(const double* __restrict__ m, const uint8_t* __restrict__ flag, double* __restrict__ y,
                        long long n) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const double r = 1.0 / m[s];
  y[s] = flag[s] ? -r : r;
}

__global__ void k_qf(const double* __restrict__ pf, const int* __restrict__ nbr, const double* __restrict__ minvf,
                     double* __restrict__ qf, long long nslots) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= nslots) return;
  const double y = minvf[nbr[s]];
  qf[s] = y > 0.0 ? pf[s] * y : 0.0;
}

__global__ void k_mass_differs(const double* __restrict__ m, long long n, int* __restrict__ differs) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && m[i] != m[0]) atomicOr(differs, 1);
}

__global__ void k_nlocf(const uint16_t* __restrict__ nloc, const int* __restrict__ nbr,
                        const uint8_t* __restrict__ flag, uint16_t* __restrict__ nlocf, long long nslots) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= nslots) return;
  nlocf[s] = static_cast<uint16_t>(nloc[s] | (flag[nbr[s]] ? 0x8000u : 0u));
}

// Bank-spread rows for the FAST particle-split chain (sweep_chain.cuh spread_slot). The chain's
// half-warps gather stencil velocities from shared memory at t.sv[d][nloc]: 16 lanes, 16 pairs of
// banks, one wavefront if the 16 indices differ mod 16 and one more per collision otherwise (ncu:
// 2.3x the ideal wavefronts with rows in slot order). Each row is regrouped into `groups` (= 2 K)
// groups of at most 16 slots, placing every slot in the group that holds the fewest slots of its
// residue (ties: the emptiest), one thread per row; group g occupies positions
// [start_g, start_g+1) of the row, header byte g = start_g (byte 0 is 0, unused groups start at
// the row's end). Writes the regrouped stencil indices (bit 15: clamped j) and pair factors. The
// regrouping changes only the order in which the FAST chain sums a row (its tolerance class).
__global__ void k_spread_rows(const long long* __restrict__ offs, const uint16_t* __restrict__ nloc,
                              const int* __restrict__ nbr, const uint8_t* __restrict__ flag,
                              const double* __restrict__ pf, int groups, uint16_t* __restrict__ nlocf,
                              double* __restrict__ pfsp, unsigned long long* __restrict__ ghdr, long long n) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long lo = offs[i];
  const int cnt = static_cast<int>(offs[i + 1] - lo);
  constexpr int kMaxRow = 128, kMaxGroups = 8;
  if (cnt > kMaxRow || cnt > 16 * groups) {  // not a row of the register chain (K <= 4): keep slot order
    for (int s = 0; s < cnt; ++s) {
      nlocf[lo + s] = static_cast<uint16_t>(nloc[lo + s] | (flag[nbr[lo + s]] ? 0x8000u : 0u));
      pfsp[lo + s] = pf[lo + s];
    }
    ghdr[i] = 0ull;
    return;
  }
  uint8_t has[kMaxGroups][16];
  uint8_t fill[kMaxGroups], grp[kMaxRow], idx[kMaxRow];
  for (int g = 0; g < kMaxGroups; ++g) {
    fill[g] = 0;
    for (int r = 0; r < 16; ++r) has[g][r] = 0;
  }
  for (int s = 0; s < cnt; ++s) {
    const int r = nloc[lo + s] & 15;
    int best = -1, best_key = 1 << 30;
    for (int g = 0; g < groups; ++g) {
      if (fill[g] >= 16) continue;
      const int key = has[g][r] * 32 + fill[g];
      if (key < best_key) {
        best_key = key;
        best = g;
      }
    }
    grp[s] = static_cast<uint8_t>(best);
    idx[s] = fill[best]++;
    ++has[best][r];
  }
  int start[kMaxGroups + 1];
  start[0] = 0;
  for (int g = 0; g < kMaxGroups; ++g) start[g + 1] = start[g] + (g < groups ? fill[g] : 0);
  unsigned long long hdr = 0ull;
  for (int g = 1; g < kMaxGroups; ++g) hdr |= static_cast<unsigned long long>(start[g]) << (8 * g);
  ghdr[i] = hdr;
  for (int s = 0; s < cnt; ++s) {
    const long long dst = lo + start[grp[s]] + idx[s];
    nlocf[dst] = static_cast<uint16_t>(nloc[lo + s] | (flag[nbr[lo + s]] ? 0x8000u : 0u));
    pfsp[dst] = pf[lo + s];
  }
}

// Dense copy of the bank-spread rows for the streamed FAST chain: row i at i * R (R = 16 * groups),
// group g at 16 g. Padding slots carry pair factor 0 (they add nothing and are never written) and
// the stencil index of their group's first slot (a broadcast in the half-warp's gather: no extra
// bank-pair wavefront); an empty group borrows the row's first slot, an empty row index 0.
__global__ void k_dense_rows(const long long* __restrict__ offs, const uint16_t* __restrict__ nlocf,
                             const double* __restrict__ pfsp, const unsigned long long* __restrict__ ghdr,
                             int groups, uint16_t* __restrict__ nld, double* __restrict__ pfd, long long n) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long lo = offs[i];
  const int cnt = static_cast<int>(offs[i + 1] - lo);
  const unsigned long long hdr = ghdr[i];
  const int R = 16 * groups;
  const long long base = i * R;
  const uint16_t row_first = cnt > 0 ? static_cast<uint16_t>(nlocf[lo] & 0x7fffu) : static_cast<uint16_t>(0);
  for (int g = 0; g < groups; ++g) {
    const int st = g == 0 ? 0 : static_cast<int>((hdr >> (8 * g)) & 0xffu);
    const int en = g + 1 < 8 ? static_cast<int>((hdr >> (8 * (g + 1))) & 0xffu) : cnt;
    const int end = g + 1 < groups ? en : cnt;  // the last group ends the row
    const uint16_t fill = end > st ? static_cast<uint16_t>(nlocf[lo + st] & 0x7fffu) : row_first;
    for (int k = 0; k < 16; ++k) {
      const bool v = st + k < end;
      nld[base + 16 * g + k] = v ? nlocf[lo + st + k] : fill;
      pfd[base + 16 * g + k] = v ? pfsp[lo + st + k] : 0.0;
    }
  }
}

// Rows re-ordered by ascending neighbour index (distinct within a row): one warp per row, each
// slot's destination is its rank in the row.
template <int D>
__global__ void k_sorted_rows(DFields f, int* __restrict__ snbr, double* __restrict__ sdw,
                              double* __restrict__ se0x, double* __restrict__ se0y, double* __restrict__ se0z) {
  const long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (i >= f.n) return;
  const long long lo = f.offs[i], hi = f.offs[i + 1];
  for (long long s = lo + lane; s < hi; s += 32) {
    const int key = f.nbr[s];
    long long rank = 0;
    for (long long t = lo; t < hi; ++t) rank += f.nbr[t] < key ? 1 : 0;
    const long long dst = lo + rank;
    snbr[dst] = key;
    sdw[dst] = f.dwdr0[s];
    se0x[dst] = f.e0[0][s];
    se0y[dst] = f.e0[1][s];
    if (D == 3) se0z[dst] = f.e0[2][s];
  }
}

template <int D>
__global__ void k_interleave_rows(DFields f, const long long* __restrict__ gbase, int* __restrict__ onbr,
                                  double* __restrict__ odw, double* __restrict__ oe0x, double* __restrict__ oe0y,
                                  double* __restrict__ oe0z) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= f.n) return;
  const long long base = gbase[i >> 5] + (i & 31), lo = f.offs[i], cnt = f.offs[i + 1] - lo;
  for (long long k = 0; k < cnt; ++k) {
    const long long src = lo + k, dst = base + 32 * k;
    onbr[dst] = f.nbr[src];
    if (D == 3 && TLSPH_TL_SLOTREC) {  // one 32-byte record per slot (tlsph.cu SlotView::load)
      *reinterpret_cast<double4*>(odw + 4 * dst) =
          make_double4(f.dwdr0[src], f.e0[0][src], f.e0[1][src], f.e0[2][src]);
      continue;
    }
    odw[dst] = f.dwdr0[src];
    oe0x[dst] = f.e0[0][src];
    oe0y[dst] = f.e0[1][src];
    if (D == 3) oe0z[dst] = f.e0[2][src];
  }
}

__global__ void k_pf_sums(DFields f) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= f.n) return;
  double a = 0.0, b = 0.0;
  for (long long s = f.offs[i]; s < f.offs[i + 1]; ++s) {
    const double p = f.pf[s];
    a = a + p;
    b = b + p * p;
  }
  f.pfsum[i] = a;
  f.pfsq[i] = b;
}

__global__ void k_cell_slot(const long long* __restrict__ cell_start, const long long* __restrict__ offs,
                            long long ncells, long long* __restrict__ out) {
  const long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c <= ncells) out[c] = offs[cell_start[c]];
}

__global__ void k_flag_in(const double* __restrict__ src, long long n, const int* __restrict__ perm, uint8_t* flag) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  flag[s] = src[perm[s]] != 0.0 ? 1 : 0;
}

__global__ void k_flag_out(double* __restrict__ dst, long long n, const int* __restrict__ perm, const uint8_t* flag) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  dst[perm[s]] = flag[s] ? 1.0 : 0.0;
}

template <int D>
__global__ void k_cell_of(DFields f, int* __restrict__ cell_of) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= f.n) return;
  double p[D];
#pragma unroll
  for (int d = 0; d < D; ++d) p[d] = f.r0[d][s];
  int c[D];
  cell_coords<D>(p, f.origin, f.cell, f.dims, c);
  cell_of[f.perm[s]] = static_cast<int>(cell_linear<D>(c, f.dims));
}

__global__ void k_row_counts_ref(DFields f, long long* __restrict__ cnt_ref) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= f.n) return;
  cnt_ref[f.perm[s]] = f.offs[s + 1] - f.offs[s];
}

template <int D>
__global__ void k_csr_to_ref(DFields f, const long long* __restrict__ off_ref, int* __restrict__ nb, double* ln,
                             double* e0, double* dw, double* pf) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= f.n) return;
  const long long src = f.offs[s], cnt = f.offs[s + 1] - src;
  const long long dst = off_ref[f.perm[s]];
  for (long long k = 0; k < cnt; ++k) {
    nb[dst + k] = f.perm[f.nbr[src + k]];
    ln[dst + k] = f.r0_len[src + k];
#pragma unroll
    for (int d = 0; d < D; ++d) e0[(dst + k) * D + d] = f.e0[d][src + k];
    dw[dst + k] = f.dwdr0[src + k];
    pf[dst + k] = f.pf[src + k];
  }
}

// Caller CSR (reference order) -> sorted rows.
__global__ void k_row_counts_sorted(DFields f, const long long* __restrict__ off_ref, long long* __restrict__ cnt) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= f.n) return;
  const int i = f.perm[s];
  cnt[s] = off_ref[i + 1] - off_ref[i];
}

template <int D>
__global__ void k_csr_from_ref(DFields f, const long long* __restrict__ off_ref, const int* __restrict__ nb,
                               const double* ln, const double* e0, const double* dw, const double* pf) {
  const long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= f.n) return;
  const int i = f.perm[s];
  const long long src = off_ref[i], cnt = off_ref[i + 1] - src, dst = f.offs[s];
  double p[D];
#pragma unroll
  for (int d = 0; d < D; ++d) p[d] = f.r0[d][s];
  int base[D];
  cell_coords<D>(p, f.origin, f.cell, f.dims, base);
  Stencil<D> st;
  stencil_segments<D>(f.cell_start, f.dims, base, st);
  for (long long k = 0; k < cnt; ++k) {
    const int j = f.rank[nb[src + k]];
    f.nbr[dst + k] = j;
    f.r0_len[dst + k] = ln[src + k];
#pragma unroll
    for (int d = 0; d < D; ++d) f.e0[d][dst + k] = e0[(src + k) * D + d];
    f.dwdr0[dst + k] = dw[src + k];
    f.pf[dst + k] = pf[src + k];
    uint16_t loc = kNoLocal;
    for (int q = 0; q < Stencil<D>::kSegs; ++q)
      if (j >= st.start[q] && j < st.start[q] + st.len[q]) {
        const long long l = st.base[q] + (j - st.start[q]);
        loc = l < kNoLocal ? static_cast<uint16_t>(l) : kNoLocal;
      }
    f.nloc[dst + k] = loc;
  }
}

// Largest padded 3^D stencil tile over the cells (sweep shared-memory sizing).
template <int D>
__global__ void k_stencil_max(DFields f, int* __restrict__ out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= f.n) return;
  double p[D];
#pragma unroll
  for (int d = 0; d < D; ++d) p[d] = f.r0[d][i];
  int c[D];
  cell_coords<D>(p, f.origin, f.cell, f.dims, c);
  Stencil<D> st;
  stencil_segments<D>(f.cell_start, f.dims, c, st);
  atomicMax(out, st.total);
}

// Sizes of the sweep's shared-memory tile: slots per cell and per particle.
__global__ void k_sweep_stats(const long long* __restrict__ cell_start, long long ncells,
                              const long long* __restrict__ offs, long long n, unsigned long long* out) {
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < ncells) {
    const long long s = offs[cell_start[t + 1]] - offs[cell_start[t]];
    atomicMax(&out[0], static_cast<unsigned long long>(s));
  }
  if (t < n) atomicMax(&out[1], static_cast<unsigned long long>(offs[t + 1] - offs[t]));
}

__global__ void k_nloc_valid(const uint16_t* nloc, long long n, int* bad) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < n && nloc[k] == kNoLocal) atomicOr(bad, 1);
}

unsigned grid_for(long long n, int block) { return static_cast<unsigned>((n + block - 1) / block); }

}  // namespace

// ====================================================================== DevSystem
DevSystem::~DevSystem() {
  for (cudaEvent_t e : halo_events)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : timer_ev)
    if (e) cudaEventDestroy(e);
  for (IpcPeer& ip : ipc_peer) ip.close();
  for (cudaEvent_t e : phase_events) cudaEventDestroy(e);
  if (stream) cudaStreamDestroy(stream);
}

DMaterial to_dmat(const tlsph_dev_material& m) {
  DMaterial d;
  d.model = m.model;
  d.lambda = m.lambda;
  d.mu = m.mu;
  d.c = m.c;
  return d;
}

DFields DevSystem::fields() const {
  DFields f{};
  f.n = n;
  f.dim = D;
  for (int d = 0; d < 3; ++d) {
    f.r0[d] = r0[d].p;
    f.r[d] = r[d].p;
    f.v[d] = v[d].p;
    f.a[d] = a[d].p;
    f.body[d] = body[d].p;
    f.e0[d] = e0[d].p;
    f.dims[d] = dims[d];
    f.origin[d] = origin[d];
  }
  for (int k = 0; k < 9; ++k) {
    f.F[k] = F[k].p;
    f.dFdt[k] = dFdt[k].p;
    f.B0[k] = B0[k].p;
  }
  f.V0 = V0.p;
  f.pbv = pbv.p;
  f.v4 = v4.p;
  f.m = m.p;
  f.minvf = minvf.p;
  f.cell_slot = cell_slot.p;
  f.fdiag = fold_diag.p;
  f.fden = fold_den.p;
  f.fy = fold_y.p;
  f.rho0 = rho0.p;
  f.rho = rho.p;
  f.flag = flag.p;
  f.perm = perm.p;
  f.rank = rank.p;
  f.offs = offs.p;
  f.nbr = nbr.p;
  f.r0_len = r0_len.p;
  f.dwdr0 = dwdr0.p;
  f.onbr = onbr.p;
  f.odw = odw.p;
  for (int d = 0; d < 3; ++d) f.oe0[d] = oe0[d].p;
  f.ogbase = ogbase.p;
  f.snbr = snbr.p;
  f.sdw = sdw.p;
  for (int d = 0; d < 3; ++d) f.se0[d] = se0[d].p;
  f.pf = pf.p;
  f.qf = qf.p;
  f.pkf = pkf.p;
  f.pfsum = pf_sum.p;
  f.peer_idx = peer_idx.p;
  f.own = own.p;
  for (int k = 0; k < 2; ++k) {
    f.peer_x[k] = peer_x[k];
    for (int d = 0; d < 3; ++d) f.peer_v[k][d] = peer_v[k][d];
  }
  f.pfsq = pf_sq.p;
  f.nloc = nloc.p;
  f.nlocf = uniform_mass ? nlocf.p : nullptr;
  f.pfsp = pfsp.p;
  f.ghdr = ghdr.p;
  f.nld = uniform_mass && dense_r > 0 ? nld.p : nullptr;
  f.pfd = pfd.p;
  f.dense_r = dense_r;
  f.minv_uniform = minv_uniform;
  f.v0_uniform = v0_uniform;
  f.cell_start = cell_start.p;
  f.cell = cutoff;
  f.has_body = has_body ? 1 : 0;
  f.contact = contact ? 1 : 0;
  for (int d = 0; d < 3; ++d) {
    f.cp_point[d] = cp_point[d];
    f.cp_normal[d] = cp_normal[d];
  }
  f.cp_k = cp_k;
  return f;
}

void DevSystem::alloc_fields() {
  const size_t N = static_cast<size_t>(n);
  for (int d = 0; d < D; ++d) {
    r0[d].alloc(N);
    r[d].alloc(N);
    v[d].alloc(N);
    a[d].alloc(N);
    body[d].alloc(N);
  }
  for (int k = 0; k < D * D; ++k) {
    F[k].alloc(N);
    dFdt[k].alloc(N);
    B0[k].alloc(N);
  }
  pbv.alloc(N * static_cast<size_t>(D == 3 ? pbv_stride<3>() : pbv_stride<2>()));
  V0.alloc(N);
  m.alloc(N);
  minvf.alloc(N);
  fold_diag.alloc(N);
  fold_den.alloc(N);
  fold_y.alloc(N);
  rho0.alloc(N);
  rho.alloc(N);
  flag.alloc(N);
  perm.alloc(N);
  rank.alloc(N);
  scal.alloc(1);
}

void DevSystem::reset_errors() {
  DScalars init{};
  for (int k = 0; k < ERR_SITES; ++k) init.err_key[k] = ~0ull;
  CK(cudaMemcpyAsync(scal.p, &init, sizeof(DScalars), cudaMemcpyHostToDevice, stream));
}

void DevSystem::init_common(int dim, size_t n_, const double* r0_h, const double* V0_h, const double* rho0_h,
                            const uint8_t* cons_h, double h_) {
  if (dim != 2 && dim != 3) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "dimension must be 2 or 3");
  if (n_ == 0) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "cell grid needs at least one particle");
  if (!(h_ > 0.0))
    throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "smoothing length must be positive, got " + std::to_string(h_));
  if (!r0_h || !V0_h || !rho0_h) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "null input array");
  D = dim;
  n = static_cast<long long>(n_);
  h = h_;
  cutoff = 2.0 * h_;  // SmoothingKernel::support_radius, runner.cpp:300-301
  CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  alloc_fields();
  reset_errors();

  // host inputs -> device
  DBuf<double> r0aos, V0d, rho0d;
  DBuf<uint8_t> consd;
  r0aos.alloc(n_ * D);
  V0d.alloc(n_);
  rho0d.alloc(n_);
  CK(cudaMemcpyAsync(r0aos.p, r0_h, n_ * D * sizeof(double), cudaMemcpyHostToDevice, stream));
  CK(cudaMemcpyAsync(V0d.p, V0_h, n_ * sizeof(double), cudaMemcpyHostToDevice, stream));
  CK(cudaMemcpyAsync(rho0d.p, rho0_h, n_ * sizeof(double), cudaMemcpyHostToDevice, stream));
  if (cons_h) {
    consd.alloc(n_);
    CK(cudaMemcpyAsync(consd.p, cons_h, n_, cudaMemcpyHostToDevice, stream));
  }

  // bounding box (neighbors.cpp:29-40)
  const unsigned nb = std::min<unsigned>(1024, grid_for(n, 256));
  DBuf<double> part;
  part.alloc(nb * 2 * D);
  DBuf<int> bad;
  bad.alloc(1);
  CK(cudaMemsetAsync(bad.p, 0, sizeof(int), stream));
  if (D == 2) k_bbox<2><<<nb, 256, 0, stream>>>(r0aos.p, n, part.p, bad.p);
  else k_bbox<3><<<nb, 256, 0, stream>>>(r0aos.p, n, part.p, bad.p);
  CK_LAUNCH("k_bbox");
  std::vector<double> hp(nb * 2 * D);
  int hbad = 0;
  CK(cudaMemcpyAsync(hp.data(), part.p, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, stream));
  CK(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
  sync();
  if (hbad) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "non-finite particle position");
  double lo[3], hi[3];
  for (int d = 0; d < D; ++d) {
    lo[d] = INFINITY;
    hi[d] = -INFINITY;
    for (unsigned b = 0; b < nb; ++b) {
      lo[d] = std::min(lo[d], hp[b * 2 * D + d]);
      hi[d] = std::max(hi[d], hp[b * 2 * D + D + d]);
    }
  }
  ncells = 1;
  for (int d = 0; d < 3; ++d) {
    if (d < D && grid_given) {
      // slab of a global grid: every local particle must lie inside it
      origin[d] = given_origin[d];
      dims[d] = given_dims[d];
      if (dims[d] < 1 || lo[d] < origin[d] || std::floor((hi[d] - origin[d]) / cutoff) >= dims[d])
        throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "particle outside the given cell grid");
    } else if (d < D) {
      origin[d] = lo[d];
      const double extent = hi[d] - lo[d];
      dims[d] = std::max(1, static_cast<int>(std::floor(extent / cutoff)) + 1);  // neighbors.cpp:45-48
    } else {
      origin[d] = 0.0;
      dims[d] = 1;
    }
    ncells *= dims[d];
  }
  if (ncells > INT_MAX) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "cell grid too large");

  // counting sort by cell key
  DBuf<int> key, count, fill, maxc;
  key.alloc(n_);
  count.alloc(static_cast<size_t>(ncells));
  fill.alloc(static_cast<size_t>(ncells));
  maxc.alloc(1);
  cell_start.alloc(static_cast<size_t>(ncells + 1));
  CK(cudaMemsetAsync(count.p, 0, ncells * sizeof(int), stream));
  CK(cudaMemsetAsync(fill.p, 0, ncells * sizeof(int), stream));
  CK(cudaMemsetAsync(maxc.p, 0, sizeof(int), stream));
  DFields f = fields();
  if (D == 2) k_cell_keys<2><<<grid_for(n, 256), 256, 0, stream>>>(r0aos.p, n, f, key.p, count.p);
  else k_cell_keys<3><<<grid_for(n, 256), 256, 0, stream>>>(r0aos.p, n, f, key.p, count.p);
  CK_LAUNCH("k_cell_keys");
  exclusive_scan<int>(count.p, ncells, cell_start.p, stream);
  k_cell_scatter<<<grid_for(n, 256), 256, 0, stream>>>(key.p, n, cell_start.p, fill.p, perm.p);
  CK_LAUNCH("k_cell_scatter");
  k_cell_sort<<<grid_for(ncells, 128), 128, 0, stream>>>(cell_start.p, ncells, perm.p, maxc.p);
  CK_LAUNCH("k_cell_sort");
  f = fields();
  if (D == 2) k_gather_init<2><<<grid_for(n, 256), 256, 0, stream>>>(f, r0aos.p, V0d.p, rho0d.p, cons_h ? consd.p : nullptr);
  else k_gather_init<3><<<grid_for(n, 256), 256, 0, stream>>>(f, r0aos.p, V0d.p, rho0d.p, cons_h ? consd.p : nullptr);
  CK_LAUNCH("k_gather_init");
  CK(cudaMemcpyAsync(&max_cell, maxc.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
  if (grid_given) {
    cell_start_h.resize(static_cast<size_t>(ncells + 1));
    CK(cudaMemcpyAsync(cell_start_h.data(), cell_start.p, cell_start_h.size() * sizeof(long long),
                       cudaMemcpyDeviceToHost, stream));
  }
  sync();
}

void DevSystem::build_neighbourhoods() {
  const double kPi = 3.14159265358979323846;
  const double sigma = (D == 2) ? 7.0 / (4.0 * kPi * h * h) : 21.0 / (16.0 * kPi * h * h * h);
  DBuf<int> counts, maxs;
  counts.alloc(static_cast<size_t>(n));
  maxs.alloc(1);
  CK(cudaMemsetAsync(maxs.p, 0, sizeof(int), stream));
  DFields f = fields();
  if (D == 2) k_nbr_count<2><<<grid_for(n, 128), 128, 0, stream>>>(f, cutoff, counts.p, maxs.p, scal.p);
  else k_nbr_count<3><<<grid_for(n, 128), 128, 0, stream>>>(f, cutoff, counts.p, maxs.p, scal.p);
  CK_LAUNCH("k_nbr_count");
  CK(cudaMemcpyAsync(&max_stencil, maxs.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
  sync();
  raise_if_failed("build_reference_neighborhoods");
  offs.alloc(static_cast<size_t>(n + 1));
  exclusive_scan<int>(counts.p, n, offs.p, stream);
  CK(cudaMemcpy(&nslots, offs.p + n, sizeof(long long), cudaMemcpyDeviceToHost));
  const size_t S = static_cast<size_t>(std::max<long long>(nslots, 1));
  nbr.alloc(S);
  r0_len.alloc(S);
  for (int d = 0; d < D; ++d) e0[d].alloc(S);
  dwdr0.alloc(S);
  pf.alloc(S);
  nloc.alloc(S);
  stencil_ok = max_stencil < 0x8000;  // staged stencil positions fit the u16 nloc
  f = fields();
  const int cap = std::max(max_stencil, 1);
  const int warps = 4;
  const size_t smem = static_cast<size_t>(warps) * cap * (4 + 4 + 2) + 16;
  if (D == 2) {
    CK(cudaFuncSetAttribute(k_nbr_fill<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k_nbr_fill<2><<<grid_for(n, warps), warps * kWarp, smem, stream>>>(f, cutoff, h, sigma, cap);
  } else {
    CK(cudaFuncSetAttribute(k_nbr_fill<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k_nbr_fill<3><<<grid_for(n, warps), warps * kWarp, smem, stream>>>(f, cutoff, h, sigma, cap);
  }
  CK_LAUNCH("k_nbr_fill");
  sync();
  compute_sweep_stats();
}

void DevSystem::refresh_minvf() {
  k_minvf<<<grid_for(n, 256), 256, 0, stream>>>(m.p, flag.p, minvf.p, n);
  CK_LAUNCH("k_minvf");
  if (nslots > 0) {
    qf.alloc(static_cast<size_t>(nslots));
    k_qf<<<grid_for(nslots, 256), 256, 0, stream>>>(pf.p, nbr.p, minvf.p, qf.p, nslots);
    CK_LAUNCH("k_qf");
  }
  // uniform masses: the streamed FAST sweep needs no per-slot or per-stencil mass data
  uniform_mass = false;
  if (n > 0 && nslots > 0 && nloc.p && stencil_ok) {
    DBuf<int> differs_d;
    differs_d.alloc(1);
    CK(cudaMemsetAsync(differs_d.p, 0, sizeof(int), stream));
    k_mass_differs<<<grid_for(n, 256), 256, 0, stream>>>(m.p, n, differs_d.p);
    CK_LAUNCH("k_mass_differs");
    int differs = 1;
    double m0 = 0.0;
    CK(cudaMemcpyAsync(&differs, differs_d.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(&m0, m.p, sizeof(double), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    if (!differs && m0 > 0.0) {
      uniform_mass = true;
      minv_uniform = 1.0 / m0;  // k_minvf's RN(1/m)
      nlocf.alloc(static_cast<size_t>(nslots));
#if TLSPH_SWEEP_SPREAD
      // rows regrouped for conflict-free gathers; the group count follows the chain's K
      // (sweep.cu launch_particle_split), known once compute_sweep_stats has the longest row
      if (max_row > 0) build_spread_rows();
#else
      k_nlocf<<<grid_for(nslots, 256), 256, 0, stream>>>(nloc.p, nbr.p, flag.p, nlocf.p, nslots);
      CK_LAUNCH("k_nlocf");
#endif
    }
  }
  fold_valid = false;  // constrained particles are marked in the fold constants
  pkf_valid = false;   // pairwise factors use the masses
}

void DevSystem::build_spread_rows() {
  if (!uniform_mass || nslots <= 0 || !nlocf.p) return;
  const int K = std::min(4, std::max(1, (max_row + kWarp - 1) / kWarp));
  pfsp.alloc(static_cast<size_t>(nslots));
  ghdr.alloc(static_cast<size_t>(n + 2));
  k_spread_rows<<<grid_for(n, 128), 128, 0, stream>>>(offs.p, nloc.p, nbr.p, flag.p, pf.p, 2 * K, nlocf.p, pfsp.p,
                                                      ghdr.p, n);
  CK_LAUNCH("k_spread_rows");
  // Dense rows for the streamed chain, opt-in (TLSPH_SWEEP_DENSE=1; measured slower than the
  // header-decoded rows: cfg4 8.28 vs 7.72 ms per sweep, cfg5-weak 14.60 vs 14.30,
  // profiles/r2e_sweep_chain_forms.md), when the device has the room (10 B per padded slot).
  static const int dense_mode = [] {
    const char* e = std::getenv("TLSPH_SWEEP_DENSE");
    return e && *e ? std::atoi(e) : 0;
  }();
  dense_r = 0;
  const bool want = dense_mode != 0;
  if (want) {
    const size_t R = static_cast<size_t>(32 * K), need = static_cast<size_t>(n) * R * 10;
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    const size_t have = (nld.p ? static_cast<size_t>(n) * R * 10 : 0) + free_b;  // a rebuild reuses its buffers
    if (have > need + (size_t(8) << 30)) {
      nld.alloc(static_cast<size_t>(n) * R);
      pfd.alloc(static_cast<size_t>(n) * R);
      k_dense_rows<<<grid_for(n, 128), 128, 0, stream>>>(offs.p, nlocf.p, pfsp.p, ghdr.p, 2 * K, nld.p, pfd.p, n);
      CK_LAUNCH("k_dense_rows");
      dense_r = static_cast<int>(R);
    }
  }
}

// ------------------------------------------------------------------ per-step re-sort (BASELINE cfg4)
// A storage permutation keyed by the *current*-position cell (the same grid as the r0 cells, out-of-
// grid positions clamped to the border cells): cell_start and the particles of each cell in ascending
// storage order. The colouring, the CSR and the sweep order stay r0-based, so
// this changes no result; with resort on, the device loop rebuilds it every step (its time is part of
// the step). Capture-safe: preallocated buffers, no host synchronisation.
void DevSystem::set_resort(bool on) {
  resort = on;
  if (!on) return;
  const size_t N = static_cast<size_t>(n), C = static_cast<size_t>(ncells);
  rs_key.alloc(N);
  rs_perm.alloc(N);
  rs_count.alloc(C);
  rs_fill.alloc(C);
  rs_start.alloc(C + 1);
  const long long tiles = (ncells + 1 + kScanTile - 1) / kScanTile;
  if (tiles + 1 > kScanTile) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "cell grid too large for the re-sort scan");
  rs_sums.alloc(static_cast<size_t>(tiles) + 1);
  rs_sums2.alloc(static_cast<size_t>(tiles) + 2);
  rs_maxc.alloc(1);
}

void DevSystem::enqueue_resort() {
  if (!resort) return;
  const DFields f = fields();
  CK(cudaMemsetAsync(rs_count.p, 0, static_cast<size_t>(ncells) * sizeof(int), stream));
  CK(cudaMemsetAsync(rs_fill.p, 0, static_cast<size_t>(ncells) * sizeof(int), stream));
  if (D == 2) k_cell_keys_current<2><<<grid_for(n, 256), 256, 0, stream>>>(f, rs_key.p, rs_count.p);
  else k_cell_keys_current<3><<<grid_for(n, 256), 256, 0, stream>>>(f, rs_key.p, rs_count.p);
  const long long n_out = ncells + 1, tiles = (n_out + kScanTile - 1) / kScanTile;
  k_scan_tile<int><<<static_cast<unsigned>(tiles), kScanThreads, 0, stream>>>(rs_count.p, ncells, rs_start.p, n_out,
                                                                              rs_sums.p);
  if (tiles > 1) {
    k_scan_tile<long long><<<1, kScanThreads, 0, stream>>>(rs_sums.p, tiles, rs_sums2.p, tiles + 1, rs_sums2.p + tiles + 1);
    k_scan_add<<<static_cast<unsigned>((n_out + 255) / 256), 256, 0, stream>>>(rs_start.p, n_out, rs_sums2.p);
  }
  k_cell_scatter<<<grid_for(n, 256), 256, 0, stream>>>(rs_key.p, n, rs_start.p, rs_fill.p, rs_perm.p);
  k_cell_sort<<<grid_for(ncells, 128), 128, 0, stream>>>(rs_start.p, ncells, rs_perm.p, rs_maxc.p);
  CK_LAUNCH("re-sort");
}

void DevSystem::current_cells(int64_t* cell_start_h, int32_t* order_ref) const {
  if (!resort) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "the per-step re-sort is off");
  std::vector<int> sorted(static_cast<size_t>(n)), pm(static_cast<size_t>(n));
  CK(cudaMemcpyAsync(cell_start_h, rs_start.p, static_cast<size_t>(ncells + 1) * sizeof(long long),
                     cudaMemcpyDeviceToHost, stream));
  CK(cudaMemcpyAsync(sorted.data(), rs_perm.p, sorted.size() * sizeof(int), cudaMemcpyDeviceToHost, stream));
  CK(cudaMemcpyAsync(pm.data(), perm.p, pm.size() * sizeof(int), cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  for (size_t k = 0; k < sorted.size(); ++k) order_ref[k] = pm[static_cast<size_t>(sorted[k])];
}

void DevSystem::refresh_v0_uniform() {
  v0_uniform = 0.0;
  if (n <= 0) return;
  DBuf<int> differs_d;
  differs_d.alloc(1);
  CK(cudaMemsetAsync(differs_d.p, 0, sizeof(int), stream));
  k_mass_differs<<<grid_for(n, 256), 256, 0, stream>>>(V0.p, n, differs_d.p);  // any array of doubles
  CK_LAUNCH("k_mass_differs");
  int differs = 1;
  double v00 = 0.0;
  CK(cudaMemcpyAsync(&differs, differs_d.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
  CK(cudaMemcpyAsync(&v00, V0.p, sizeof(double), cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  if (!differs && v00 > 0.0) v0_uniform = v00;
}

// Slot arrays interleaved by groups of 32 particles for the ORDERED neighbour passes (one thread
// per particle walks its row in slot order; this layout makes a warp's loads of slot k contiguous).
// Large bodies (n >= 65,536) run the neighbour passes of BOTH modes as one thread per particle
// summing in slot order over this layout: bit-exact (the ORDERED arithmetic) and faster than the
// eight-lanes-per-particle FAST kernels (cfg3 elastic step 1.040 -> 0.987 ms). Small bodies keep
// the row-contiguous layout (few warps per SM: a thread's own row in one cache line wins; cfg1,
// 16,000 particles: 49 vs 66 ms of ORDERED elastic kernels per 2,000 steps) and FAST's eight lanes.
void DevSystem::build_ordered_rows() {
  if (nslots <= 0 || n < 65536) return;
  std::vector<long long> off(static_cast<size_t>(n) + 1);
  CK(cudaMemcpyAsync(off.data(), offs.p, off.size() * sizeof(long long), cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  const long long groups = (n + 31) / 32;
  std::vector<long long> gb(static_cast<size_t>(groups) + 1, 0);
  for (long long g = 0; g < groups; ++g) {
    long long mx = 0;
    for (long long i = 32 * g; i < std::min<long long>(n, 32 * g + 32); ++i) mx = std::max(mx, off[i + 1] - off[i]);
    gb[g + 1] = gb[g] + 32 * mx;
  }
  const size_t total = static_cast<size_t>(std::max<long long>(gb[groups], 1));
  ogbase.alloc(gb.size());
  CK(cudaMemcpyAsync(ogbase.p, gb.data(), gb.size() * sizeof(long long), cudaMemcpyHostToDevice, stream));
  onbr.alloc(total);
  if (D == 3 && TLSPH_TL_V4) v4.alloc(4 * static_cast<size_t>(n));
  if (D == 3 && TLSPH_TL_SLOTREC) {
    odw.alloc(4 * total);  // (dW/dr0, e0) records
  } else {
    odw.alloc(total);
    for (int d = 0; d < D; ++d) oe0[d].alloc(total);
  }
  const DFields f = fields();
  if (D == 2)
    k_interleave_rows<2><<<grid_for(n, 256), 256, 0, stream>>>(f, ogbase.p, onbr.p, odw.p, oe0[0].p, oe0[1].p, nullptr);
  else
    k_interleave_rows<3><<<grid_for(n, 256), 256, 0, stream>>>(f, ogbase.p, onbr.p, odw.p, oe0[0].p, oe0[1].p,
                                                               oe0[2].p);
  CK_LAUNCH("k_interleave_rows");
  sync();
}

void DevSystem::compute_sweep_stats() {
  build_ordered_rows();  // large bodies: both modes' neighbour passes (slot order, coalesced)
  refresh_minvf();
  refresh_v0_uniform();
  if (nslots > 0 && !onbr.p) {  // small bodies: FAST passes on eight lanes per particle, rows by neighbour
    const size_t S = static_cast<size_t>(nslots);
    snbr.alloc(S);
    sdw.alloc(S);
    for (int d = 0; d < D; ++d) se0[d].alloc(S);
    const DFields f = fields();
    const unsigned grid = static_cast<unsigned>((n * 32 + 255) / 256);
    if (D == 2) k_sorted_rows<2><<<grid, 256, 0, stream>>>(f, snbr.p, sdw.p, se0[0].p, se0[1].p, nullptr);
    else k_sorted_rows<3><<<grid, 256, 0, stream>>>(f, snbr.p, sdw.p, se0[0].p, se0[1].p, se0[2].p);
    CK_LAUNCH("k_sorted_rows");
  }
  pf_sum.alloc(static_cast<size_t>(n));
  pf_sq.alloc(static_cast<size_t>(n));
  k_pf_sums<<<grid_for(n, 256), 256, 0, stream>>>(fields());
  CK_LAUNCH("k_pf_sums");
  cell_slot.alloc(static_cast<size_t>(ncells + 1));
  k_cell_slot<<<grid_for(ncells + 1, 256), 256, 0, stream>>>(cell_start.p, offs.p, ncells, cell_slot.p);
  CK_LAUNCH("k_cell_slot");
  DBuf<unsigned long long> out;
  out.alloc(2);
  CK(cudaMemsetAsync(out.p, 0, 2 * sizeof(unsigned long long), stream));
  const long long m = std::max(ncells, n);
  k_sweep_stats<<<grid_for(m, 256), 256, 0, stream>>>(cell_start.p, ncells, offs.p, n, out.p);
  CK_LAUNCH("k_sweep_stats");
  unsigned long long h[2] = {0, 0};
  CK(cudaMemcpyAsync(h, out.p, sizeof(h), cudaMemcpyDeviceToHost, stream));
  sync();
  max_cell_slots = static_cast<long long>(h[0]);
  max_row = static_cast<int>(h[1]);
#if TLSPH_SWEEP_SPREAD
  build_spread_rows();  // refresh_minvf above ran before the longest row was known
#endif
  build_colour_lists();
}

void DevSystem::load_csr(const int64_t* offsets, const int32_t* neighbor, const double* r0_len_h, const double* e0_h,
                         const double* dwdr0_h, const double* pf_h) {
  const size_t N = static_cast<size_t>(n);
  nslots = offsets[N];
  const size_t S = static_cast<size_t>(std::max<long long>(nslots, 1));
  DBuf<long long> off_ref, cnt;
  DBuf<int> nb_ref;
  DBuf<double> ln_ref, e0_ref, dw_ref, pf_ref;
  off_ref.alloc(N + 1);
  nb_ref.alloc(S);
  ln_ref.alloc(S);
  e0_ref.alloc(S * D);
  dw_ref.alloc(S);
  pf_ref.alloc(S);
  CK(cudaMemcpyAsync(off_ref.p, offsets, (N + 1) * sizeof(long long), cudaMemcpyHostToDevice, stream));
  if (nslots > 0) {
    copy_to_device(nb_ref.p, neighbor, nslots * sizeof(int), stream);
    copy_to_device(ln_ref.p, r0_len_h, nslots * sizeof(double), stream);
    copy_to_device(e0_ref.p, e0_h, nslots * D * sizeof(double), stream);
    copy_to_device(dw_ref.p, dwdr0_h, nslots * sizeof(double), stream);
    copy_to_device(pf_ref.p, pf_h, nslots * sizeof(double), stream);
  }
  cnt.alloc(N);
  offs.alloc(N + 1);
  DFields f = fields();
  k_row_counts_sorted<<<grid_for(n, 256), 256, 0, stream>>>(f, off_ref.p, cnt.p);
  CK_LAUNCH("k_row_counts_sorted");
  exclusive_scan<long long>(cnt.p, n, offs.p, stream);
  nbr.alloc(S);
  r0_len.alloc(S);
  for (int d = 0; d < D; ++d) e0[d].alloc(S);
  dwdr0.alloc(S);
  pf.alloc(S);
  nloc.alloc(S);
  // staged-stencil size for the sweep kernels
  {
    DBuf<int> maxs;
    maxs.alloc(1);
    CK(cudaMemsetAsync(maxs.p, 0, sizeof(int), stream));
    f = fields();
    if (D == 2) k_stencil_max<2><<<grid_for(n, 128), 128, 0, stream>>>(f, maxs.p);
    else k_stencil_max<3><<<grid_for(n, 128), 128, 0, stream>>>(f, maxs.p);
    CK_LAUNCH("k_stencil_max");
    CK(cudaMemcpyAsync(&max_stencil, maxs.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
    sync();
  }
  f = fields();
  if (D == 2) k_csr_from_ref<2><<<grid_for(n, 128), 128, 0, stream>>>(f, off_ref.p, nb_ref.p, ln_ref.p, e0_ref.p, dw_ref.p, pf_ref.p);
  else k_csr_from_ref<3><<<grid_for(n, 128), 128, 0, stream>>>(f, off_ref.p, nb_ref.p, ln_ref.p, e0_ref.p, dw_ref.p, pf_ref.p);
  CK_LAUNCH("k_csr_from_ref");
  DBuf<int> bad;
  bad.alloc(1);
  CK(cudaMemsetAsync(bad.p, 0, sizeof(int), stream));
  if (nslots > 0) {
    k_nloc_valid<<<grid_for(nslots, 256), 256, 0, stream>>>(nloc.p, nslots, bad.p);
    CK_LAUNCH("k_nloc_valid");
  }
  int hbad = 0;
  CK(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
  sync();
  stencil_ok = (hbad == 0) && max_stencil < 0x8000;
  compute_sweep_stats();
}

namespace {
struct FieldSpec {
  int comps;
  std::vector<double*> ptrs;
  FieldPtrs pack() const {
    FieldPtrs fp{};
    for (size_t k = 0; k < ptrs.size() && k < 9; ++k) fp.p[k] = ptrs[k];
    return fp;
  }
};
}  // namespace

static FieldSpec field_spec(const DevSystem& s, int field) {
  FieldSpec fs;
  auto vec = [&](const DBuf<double>* arr) {
    fs.comps = s.D;
    for (int d = 0; d < s.D; ++d) fs.ptrs.push_back(arr[d].p);
  };
  auto mat = [&](const DBuf<double>* arr) {
    fs.comps = s.D * s.D;
    for (int k = 0; k < s.D * s.D; ++k) fs.ptrs.push_back(arr[k].p);
  };
  auto sc = [&](const DBuf<double>& arr) {
    fs.comps = 1;
    fs.ptrs.push_back(arr.p);
  };
  switch (field) {
    case TLSPH_FIELD_R0: vec(s.r0); break;
    case TLSPH_FIELD_R: vec(s.r); break;
    case TLSPH_FIELD_V: vec(s.v); break;
    case TLSPH_FIELD_A: vec(s.a); break;
    case TLSPH_FIELD_BODY: vec(s.body); break;
    case TLSPH_FIELD_F: mat(s.F); break;
    case TLSPH_FIELD_DFDT: mat(s.dFdt); break;
    case TLSPH_FIELD_B0: mat(s.B0); break;
    case TLSPH_FIELD_V0: sc(s.V0); break;
    case TLSPH_FIELD_M: sc(s.m); break;
    case TLSPH_FIELD_RHO0: sc(s.rho0); break;
    case TLSPH_FIELD_RHO: sc(s.rho); break;
    default: throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "unknown field id " + std::to_string(field));
  }
  return fs;
}

void DevSystem::set_field(int field, const double* host) {
  if (!host) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "null host array");
  const size_t N = static_cast<size_t>(n);
  if (field == TLSPH_FIELD_CONSTRAINED) {
    tmp.alloc(N);
    copy_to_device(tmp.p, host, N * sizeof(double), stream);
    k_flag_in<<<grid_for(n, 256), 256, 0, stream>>>(tmp.p, n, perm.p, flag.p);
    CK_LAUNCH("k_flag_in");
    refresh_minvf();
    sync();
    return;
  }
  if (field == TLSPH_FIELD_R0)
    throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "r0 is fixed at construction (the cell grid is built from it)");
  FieldSpec fs = field_spec(*this, field);
  tmp.alloc(N * fs.comps);
  copy_to_device(tmp.p, host, N * fs.comps * sizeof(double), stream);
  g_h2d_bytes += N * fs.comps * sizeof(double);
  k_aos_to_soa<<<grid_for(n, 256), 256, 0, stream>>>(tmp.p, fs.comps, n, perm.p, fs.pack());
  CK_LAUNCH("k_aos_to_soa");
  if (field == TLSPH_FIELD_BODY) has_body = true;
  if (field == TLSPH_FIELD_M) {
    refresh_minvf();
    fold_valid = false;  // diag = sum b - m_i
  }
  if (field == TLSPH_FIELD_V0) refresh_v0_uniform();
  sync();
}

void DevSystem::get_field(int field, double* host) const {
  if (!host) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "null host array");
  const size_t N = static_cast<size_t>(n);
  auto* self = const_cast<DevSystem*>(this);
  if (field == TLSPH_FIELD_CONSTRAINED) {
    self->tmp.alloc(N);
    k_flag_out<<<grid_for(n, 256), 256, 0, stream>>>(tmp.p, n, perm.p, flag.p);
    CK_LAUNCH("k_flag_out");
    copy_to_host(host, tmp.p, N * sizeof(double), stream);
    sync();
    return;
  }
  FieldSpec fs = field_spec(*this, field);
  self->tmp.alloc(N * fs.comps);
  k_soa_to_aos<<<grid_for(n, 256), 256, 0, stream>>>(tmp.p, fs.comps, n, perm.p, fs.pack());
  CK_LAUNCH("k_soa_to_aos");
  copy_to_host(host, tmp.p, N * fs.comps * sizeof(double), stream);
  sync();
}

void DevSystem::put_record(int field, const void* host, int layout, bool only_if_changed, int* changed) {
  if (!host && field == TLSPH_FIELD_BODY) {  // no body term (ExternalAccel::body empty)
    if (changed) *changed = has_body ? 1 : 0;
    if (has_body)  // the kernels always add body[i]: zero it once when the term goes away
      for (int d = 0; d < D; ++d) CK(cudaMemsetAsync(body[d].p, 0, static_cast<size_t>(n) * sizeof(double), stream));
    has_body = false;
    sync();
    return;
  }
  if (!host) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "null host array");
  if (layout != 0 && layout != 1) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "record layout must be 0 or 1");
  const size_t N = static_cast<size_t>(n);
  if (changed) *changed = 1;
  DBuf<int>& differs = flag_buf;
  differs.alloc(1);
  auto any_differs = [&] {
    int h = 0;
    CK(cudaMemcpyAsync(&h, differs.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
    sync();
    return h != 0;
  };
  if (field == TLSPH_FIELD_CONSTRAINED) {
    tmp.alloc((N + 7) / 8);
    auto* staged = reinterpret_cast<uint8_t*>(tmp.p);
    copy_to_device(staged, host, N, stream);
    g_h2d_bytes += N;
    if (only_if_changed) {
      CK(cudaMemsetAsync(differs.p, 0, sizeof(int), stream));
      k_flags_in<<<grid_for(n, 256), 256, 0, stream>>>(staged, n, perm.p, flag.p, differs.p);
      CK_LAUNCH("k_flags_in");
      if (!any_differs()) {
        if (changed) *changed = 0;
        return;
      }
    }
    k_flags_in<<<grid_for(n, 256), 256, 0, stream>>>(staged, n, perm.p, flag.p, nullptr);
    CK_LAUNCH("k_flags_in");
    refresh_minvf();
    sync();
    return;
  }
  FieldSpec fs = field_spec(*this, field == TLSPH_FIELD_R0 ? TLSPH_FIELD_R0 : field);
  const int cm = layout == 1 && fs.comps == D * D ? D : 0;
  tmp.alloc(N * fs.comps);
  copy_to_device(tmp.p, host, N * fs.comps * sizeof(double), stream);
  g_h2d_bytes += N * fs.comps * sizeof(double);
  if (only_if_changed || field == TLSPH_FIELD_R0) {
    CK(cudaMemsetAsync(differs.p, 0, sizeof(int), stream));
    k_records_differ<<<grid_for(n, 256), 256, 0, stream>>>(tmp.p, fs.comps, cm, n, perm.p, fs.pack(), differs.p);
    CK_LAUNCH("k_records_differ");
    if (!any_differs()) {
      if (changed) *changed = 0;
      return;
    }
    if (field == TLSPH_FIELD_R0)
      throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "r0 is fixed at construction (the cell grid is built from it)");
  }
  k_records_in<<<grid_for(n, 256), 256, 0, stream>>>(tmp.p, fs.comps, cm, n, perm.p, fs.pack());
  CK_LAUNCH("k_records_in");
  if (field == TLSPH_FIELD_BODY) has_body = true;
  if (field == TLSPH_FIELD_M) {
    refresh_minvf();
    fold_valid = false;  // diag = sum b - m_i
  }
  if (field == TLSPH_FIELD_V0) refresh_v0_uniform();
  sync();
}

void DevSystem::take_record(int field, void* host, int layout) const {
  if (!host) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "null host array");
  if (layout != 0 && layout != 1) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "record layout must be 0 or 1");
  const size_t N = static_cast<size_t>(n);
  auto* self = const_cast<DevSystem*>(this);
  if (field == TLSPH_FIELD_CONSTRAINED) {
    self->tmp.alloc((N + 7) / 8);
    auto* staged = reinterpret_cast<uint8_t*>(tmp.p);
    k_flags_out<<<grid_for(n, 256), 256, 0, stream>>>(staged, n, perm.p, flag.p);
    CK_LAUNCH("k_flags_out");
    copy_to_host(host, staged, N, stream);
    g_d2h_bytes += N;
    sync();
    return;
  }
  FieldSpec fs = field_spec(*this, field);
  const int cm = layout == 1 && fs.comps == D * D ? D : 0;
  self->tmp.alloc(N * fs.comps);
  k_records_out<<<grid_for(n, 256), 256, 0, stream>>>(tmp.p, fs.comps, cm, n, perm.p, fs.pack());
  CK_LAUNCH("k_records_out");
  copy_to_host(host, tmp.p, N * fs.comps * sizeof(double), stream);
  g_d2h_bytes += N * fs.comps * sizeof(double);
  sync();
}

void DevSystem::grid_cells(int32_t* cell_of, int64_t* cell_start_h, int32_t* cell_particles) const {
  const size_t N = static_cast<size_t>(n);
  DBuf<int> co;
  co.alloc(N);
  DFields f = fields();
  if (D == 2) k_cell_of<2><<<grid_for(n, 256), 256, 0, stream>>>(f, co.p);
  else k_cell_of<3><<<grid_for(n, 256), 256, 0, stream>>>(f, co.p);
  CK_LAUNCH("k_cell_of");
  if (cell_of) copy_to_host(cell_of, co.p, N * sizeof(int), stream);
  if (cell_start_h)
    CK(cudaMemcpyAsync(cell_start_h, cell_start.p, (ncells + 1) * sizeof(long long), cudaMemcpyDeviceToHost, stream));
  if (cell_particles) copy_to_host(cell_particles, perm.p, N * sizeof(int), stream);
  sync();
}

void DevSystem::get_neighborhood(int64_t* offsets, int32_t* neighbor, double* r0_len_h, double* e0_h,
                                 double* dwdr0_h, double* pf_h) const {
  const size_t N = static_cast<size_t>(n);
  const size_t S = static_cast<size_t>(std::max<long long>(nslots, 1));
  DBuf<long long> cnt, off_ref;
  cnt.alloc(N);
  off_ref.alloc(N + 1);
  DFields f = fields();
  k_row_counts_ref<<<grid_for(n, 256), 256, 0, stream>>>(f, cnt.p);
  CK_LAUNCH("k_row_counts_ref");
  exclusive_scan<long long>(cnt.p, n, off_ref.p, stream);
  if (!neighbor && !r0_len_h && !e0_h && !dwdr0_h && !pf_h) {  // row offsets only
    if (offsets) CK(cudaMemcpyAsync(offsets, off_ref.p, (N + 1) * sizeof(long long), cudaMemcpyDeviceToHost, stream));
    sync();
    return;
  }
  DBuf<int> nb;
  DBuf<double> ln, e, dw, p;
  nb.alloc(S);
  ln.alloc(S);
  e.alloc(S * D);
  dw.alloc(S);
  p.alloc(S);
  if (D == 2) k_csr_to_ref<2><<<grid_for(n, 128), 128, 0, stream>>>(f, off_ref.p, nb.p, ln.p, e.p, dw.p, p.p);
  else k_csr_to_ref<3><<<grid_for(n, 128), 128, 0, stream>>>(f, off_ref.p, nb.p, ln.p, e.p, dw.p, p.p);
  CK_LAUNCH("k_csr_to_ref");
  if (offsets) CK(cudaMemcpyAsync(offsets, off_ref.p, (N + 1) * sizeof(long long), cudaMemcpyDeviceToHost, stream));
  if (nslots > 0) {
    if (neighbor) copy_to_host(neighbor, nb.p, nslots * sizeof(int), stream);
    if (r0_len_h) copy_to_host(r0_len_h, ln.p, nslots * sizeof(double), stream);
    if (e0_h) copy_to_host(e0_h, e.p, nslots * D * sizeof(double), stream);
    if (dwdr0_h) copy_to_host(dwdr0_h, dw.p, nslots * sizeof(double), stream);
    if (pf_h) copy_to_host(pf_h, p.p, nslots * sizeof(double), stream);
  }
  sync();
}

// Translates recorded device errors into the reference's exception text.
void DevSystem::raise_if_failed(const char* context) {
  DScalars hs;
  CK(cudaMemcpyAsync(&hs, scal.p, sizeof(DScalars), cudaMemcpyDeviceToHost, stream));
  sync();
  if (!hs.failed) return;
  for (int site = 0; site < ERR_SITES; ++site) {
    const unsigned long long key = hs.err_key[site];
    if (key == ~0ull) continue;
    std::string msg;
    tlsph_status st = TLSPH_ERR_INTERNAL;
    switch (site) {
      case ERR_DENSITY_PRE:
      case ERR_MOMENTUM:
      case ERR_DENSITY_POST:
        st = TLSPH_ERR_INVERTED_ELEMENT;
        msg = "inverted element: det(F) <= 0 for particle " + std::to_string(key);
        break;
      case ERR_NAN:
        st = TLSPH_ERR_NUMERICAL_FAILURE;
        msg = "NaN detected at step " + std::to_string(hs.err_step) + ", particle " + std::to_string(key);
        break;
      case ERR_DEGENERATE:
        st = TLSPH_ERR_DEGENERATE_GEOMETRY;
        msg = "degenerate neighborhood: correction matrix of particle " + std::to_string(key) +
              " is singular or ill-conditioned";
        break;
      case ERR_COINCIDENT: {
        st = TLSPH_ERR_DEGENERATE_GEOMETRY;
        const long long ri = static_cast<long long>(key >> 32);
        const int s = static_cast<int>((key >> 24) & 0xFF);
        const long long k = static_cast<long long>(key & 0xFFFFFF);
        // decode the partner: the s-th stencil cell of ri, k-th particle in it
        int si = 0;
        CK(cudaMemcpy(&si, rank.p + ri, sizeof(int), cudaMemcpyDeviceToHost));
        double p[3] = {0, 0, 0};
        for (int d = 0; d < D; ++d) CK(cudaMemcpy(&p[d], r0[d].p + si, sizeof(double), cudaMemcpyDeviceToHost));
        int c[3] = {0, 0, 0};
        int rem = s;
        for (int d = 0; d < D; ++d) {
          int idx = static_cast<int>(std::floor((p[d] - origin[d]) / cutoff));
          idx = std::clamp(idx, 0, dims[d] - 1);
          c[d] = idx + (rem % 3) - 1;
          rem /= 3;
        }
        long long lin = c[D - 1];
        for (int d = D - 2; d >= 0; --d) lin = lin * dims[d] + c[d];
        long long start = 0;
        CK(cudaMemcpy(&start, cell_start.p + lin, sizeof(long long), cudaMemcpyDeviceToHost));
        int rj = 0;
        CK(cudaMemcpy(&rj, perm.p + start + k, sizeof(int), cudaMemcpyDeviceToHost));
        msg = "coincident particles " + std::to_string(ri) + " and " + std::to_string(rj) +
              " in reference configuration";
        break;
      }
      default:
        msg = std::string("device failure in ") + context;
    }
    reset_errors();
    throw DevError(st, msg);
  }
}

}  // namespace tlsph_cuda
