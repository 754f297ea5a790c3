// The FAST particle-split Gauss-Seidel chain of one cell, run by one warp
// (damping.cpp:53-89 particle_split_update, applied in cell order as
// neighbors.cpp:143-174 block_sweep does). Shared by k_sweep_fast (sweep.cu)
// and the microbenchmark tools/chain_fast.cu.
//
// Lane l owns slots l, l+32, ... (K per lane) of the current particle for all
// D velocity components. Reassociated update (FAST tolerance class): with
// w = v_j - v_i, Y = v_j + bm w and C = -bm (diag + b),
//   v_j' = v_j - bm (v_i + diag rate - (v_j - b rate)) = Y + C rate,
// so one FMA per slot follows the residual reduction on the chain (rate = residual * y with
// y = RN(1 / denominator); TLSPH_CHAIN_NORATE folds y into C and diag when they are formed, so the
// FMA acts on the reduced residual itself). The D residuals are summed over the warp by two fp64
// MMAs per component and no shuffle (warp_sum_vec_mma2). Y is formed from w (not as
// (1 + bm) v_j - bm v_i): a uniform velocity field (w = 0, rate = 0) is left exactly unchanged, as
// in the reference's order -- the sweep amplifies any non-uniformity when eta~ dt is large (the
// falling-ball case), so FAST must not create one.
//
// Software pipeline. Everything but the stencil velocities is static during
// the chain, so the slot metadata of the next particle is loaded while the
// current one runs: (A) its neighbour indices, pair factors and per-slot mass
// factors pair_factor / m_j (precomputed per body, so no gather through the
// neighbour index), issued at the top of the iteration; (C) its fold
// constants; (D) the derived coefficients, formed after the scatter. Row
// extents are read two particles ahead. A constrained particle (NaN
// diagonal) or one without neighbours (damping.cpp:54, :151) runs the same
// code with its writes disabled, so the loop has no data-dependent branch.
#pragma once
// TLSPH_CHAIN_NORATE (default 1): 1/denominator folded into the slot coefficients when they are
// formed (c y and diag y), so the scatter is one FMA on the reduced residual, without the rate
// product on the chain (another rounding of the FAST class; 0 = the former rate form).
#ifndef TLSPH_CHAIN_NORATE
#define TLSPH_CHAIN_NORATE 1
#endif
// Y of the FAST update (see below): v_j + bm (v_j - v_i) (default), or the former
// (1 + bm) v_j - bm v_i (TLSPH_Y_FORM=2: not exact for uniform fields; A/B only)
// streamed chain: Y formed at the scatter (1) or before the reduction (0)
#ifndef TLSPH_Y_LATE
#define TLSPH_Y_LATE 1
#endif
#if defined(TLSPH_Y_FORM) && TLSPH_Y_FORM == 2
#define TLSPH_Y(u, d) __fma_rn(1.0 + bmq[u], vq[u][d], -bmq[u] * vi[d])
#elif defined(TLSPH_Y_FORM) && TLSPH_Y_FORM == 3
#define TLSPH_Y(u, d) __dadd_rn(vq[u][d], __dmul_rn(bmq[u], vq[u][d] - vi[d]))
#else
#define TLSPH_Y(u, d) __fma_rn(bmq[u], vq[u][d] - vi[d], vq[u][d])
#endif
#include <cstdint>

// Bank-spread rows (UNI chains): the sweep's own copy of a row's slots (stencil index, pair
// factor) is regrouped so that the 16 lanes of a half-warp gather from 16 distinct shared-memory
// bank pairs (state.cu k_spread_rows); a per-particle header gives the group extents.
#ifndef TLSPH_SWEEP_SPREAD
#define TLSPH_SWEEP_SPREAD 1
#endif

// A/B knob (measured, rejected: profiles/r2e_sweep_idle_lanes.md). Idle lanes (no slot in this
// iteration, pair factor 0) gather particle i's own entry; with the knob on they gather the stencil
// entry of lane 0 of their half-warp instead, so that the half-warp's 64-bit shared-memory request
// carries no second address in i's bank pair. The shuffle per slot iteration that forms the index
// costs more than the saved wavefronts: cfg2 0.636 -> 0.673 ms, cfg4 8.95 -> 9.88, cfg5-weak 15.9 -> 17.6.
#ifndef TLSPH_SWEEP_IDLE_BCAST
#define TLSPH_SWEEP_IDLE_BCAST 0
#endif

namespace tlsph_cuda {

// Stencil index an idle lane gathers (its result is multiplied by b = 0 and never scattered).
__device__ __forceinline__ int idle_lane_index(int j, bool idle, int lane) {
#if TLSPH_SWEEP_IDLE_BCAST
  const int j0 = __shfl_sync(0xffffffffu, j, lane & 16);
  return idle ? j0 : j;
#else
  (void)idle;
  (void)lane;
  return j;
#endif
}

// Slot of this lane in iteration u of a bank-spread row: half-warp h = lane / 16 reads group
// g = 2u + h, positions [start_g, start_g+1) of the row. Header byte g = start_g (byte 0 = 0;
// groups the row does not use start at cnt).
template <int K>
__device__ __forceinline__ void spread_slot(unsigned long long hdr, int cnt, int lane, int u, int& s, bool& v) {
  const unsigned lo = static_cast<unsigned>(hdr), hi = static_cast<unsigned>(hdr >> 32);
  const unsigned g = 2u * static_cast<unsigned>(u) + (static_cast<unsigned>(lane) >> 4);
  // selector nibbles 1-3 are 0: they pick byte 0 of the header, which is zero
  const int st = static_cast<int>(__byte_perm(lo, hi, g));
  int en = static_cast<int>(__byte_perm(lo, hi, (g + 1) & 7));
  if (2 * u + 2 >= 8 && (lane >> 4)) en = cnt;  // group 7 ends the row
  s = st + (lane & 15);
  v = s < en;
}

template <int D>
struct ChainTile {
  double* sv[D];          // staged stencil velocities
  const double* pf;       // the cell's pair factors, cell-relative slot index
  const double* qf;       // pair_factor / m_j per slot (0: clamped j, never written)
  const uint16_t* nl;     // the cell's stencil-local neighbour indices
  const double* smf;      // fast_chain_stream: staged stencil signed RN(1/m) (negative: clamped)
  double minv;            // fast_chain_stream<UNI>: the uniform RN(1/m); nl carries bit 15 = clamped j
  const long long* offs;  // offs[p] - s0 = cell-relative first slot of particle p
  const unsigned long long* hdr;  // bank-spread rows: group extents per particle (spread_slot)
  const uint16_t* nlb;    // fast_chain_stream: the body's slot arrays (index s0u + cell-relative slot)
  const double* pfb;
  unsigned s0u;
  long long s0;
  const double* diag;     // per-particle fold constants (NaN: constrained particle)
  const double* y;        // RN(1 / denominator)
  int lbase;              // tile index of the cell's first particle
  int np;
  int forward;
  double kb;              // b = kb * pair_factor
};

// Sum of D doubles over the warp, result in every lane. Transposing
// butterfly: the first levels exchange half of the remaining components
// (lane bit 4 picks components {0,1} or {2,3}, bit 3 one of the pair), so
// after two levels each lane carries one component and the last three levels
// are a plain butterfly; one broadcast per component follows. 18 32-bit
// shuffles for D = 3 instead of 30, and every level depends on all
// components, so the reductions cannot be serialised by the scheduler.
template <int D>
__device__ __forceinline__ void warp_sum_vec(double (&x)[D], int lane) {
  static_assert(D == 2 || D == 3, "D");
  constexpr unsigned kAll = 0xffffffffu;
  const bool b4 = lane & 16, b3 = lane & 8;
  double c;
  if constexpr (D == 3) {
    const double a0 = b4 ? x[0] : x[2], a1 = b4 ? x[1] : 0.0;  // sent
    const double k0 = b4 ? x[2] : x[0], k1 = b4 ? 0.0 : x[1];  // kept
    const double r0 = __shfl_xor_sync(kAll, a0, 16), r1 = __shfl_xor_sync(kAll, a1, 16);
    const double h0 = k0 + r0, h1 = k1 + r1;  // components 2 b4, 2 b4 + 1
    const double r = __shfl_xor_sync(kAll, b3 ? h0 : h1, 8);
    c = (b3 ? h1 : h0) + r;  // component 2 b4 + b3
  } else {
    const double r = __shfl_xor_sync(kAll, b4 ? x[0] : x[1], 16);
    c = (b4 ? x[1] : x[0]) + r;  // component b4
  }
#pragma unroll
  for (int o = D == 3 ? 4 : 8; o > 0; o >>= 1) c += __shfl_xor_sync(kAll, c, o);
#pragma unroll
  for (int d = 0; d < D; ++d) x[d] = __shfl_sync(kAll, c, D == 3 ? 8 * d : 16 * d);
}

// UNI (uniform masses): no per-slot mass factors; qf = pair_factor * RN(1/m)
// unless bit 15 of the stencil index marks a clamped j (exactly the stored qf).
// The same sum through the fp64 tensor-core MMA (mma.sync m8n8k4, B = ones): one MMA per
// component sums each group of four lanes (lane 4r+k supplies A[r][k]; every lane of group r
// receives the group sum), then a three-level xor butterfly adds the eight group sums. Dependent
// latency ~185 cycles against ~233 for the shuffle tree (tools/dmma_probe.cu); the summation order
// differs (FAST class).
// TLSPH_SWEEP_MMA_SUM: 0 = shuffle tree, 1 = one MMA + three butterfly levels, 2 (default) = two
// MMAs and no shuffle (warp_sum_vec_mma2; same-box A/B against 1, ms per sweep: cfg2 0.636 -> 0.597,
// cfg3 1.088 -> 1.070, cfg4 8.95 -> 8.65, cfg5-weak 15.89 -> 15.42; profiles/r2e_sweep_mma2.md).
#ifndef TLSPH_SWEEP_MMA_SUM
#define TLSPH_SWEEP_MMA_SUM 2
#endif
template <int D>
__device__ __forceinline__ void warp_sum_vec_mma(double (&x)[D]) {
  constexpr unsigned kAll = 0xffffffffu;
  double r[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    double unused;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
                 : "=d"(r[d]), "=d"(unused)
                 : "d"(x[d]), "d"(1.0), "d"(0.0), "d"(0.0));
  }
#pragma unroll
  for (int o = 4; o < 32; o <<= 1)
#pragma unroll
    for (int d = 0; d < D; ++d) r[d] += __shfl_xor_sync(kAll, r[d], o);
#pragma unroll
  for (int d = 0; d < D; ++d) x[d] = r[d];
}

// The whole sum by two MMAs and no shuffle (TLSPH_SWEEP_MMA_SUM=2). First MMA with A = ones and the
// lanes' values as B (lane 4n+k supplies B[k][n]): D[m][n] = G_n, the sum of lane group n, and lane
// 4r+k receives G_2k and G_2k+1; it adds them. Second MMA with those pair sums as A (lane 4r+k
// supplies A[r][k]) and B = ones: D[r][n] = sum_k (G_2k + G_2k+1), the total, in every lane.
template <int D>
__device__ __forceinline__ void warp_sum_vec_mma2(double (&x)[D]) {
  double p[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    double c0, c1;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
                 : "=d"(c0), "=d"(c1)
                 : "d"(1.0), "d"(x[d]), "d"(0.0), "d"(0.0));
    p[d] = c0 + c1;
  }
#pragma unroll
  for (int d = 0; d < D; ++d) {
    double unused;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
                 : "=d"(x[d]), "=d"(unused)
                 : "d"(p[d]), "d"(1.0), "d"(0.0), "d"(0.0));
  }
}

template <int D>
__device__ __forceinline__ void chain_sum(double (&x)[D], int lane) {
  if (TLSPH_SWEEP_MMA_SUM == 2) warp_sum_vec_mma2<D>(x);
  else if (TLSPH_SWEEP_MMA_SUM) warp_sum_vec_mma<D>(x);
  else warp_sum_vec<D>(x, lane);
}

template <int D, int K, bool SHUF = true, bool SCATTER = true, bool UNI = false, bool SPREAD = false>
__device__ __forceinline__ void fast_chain(const ChainTile<D>& t, int lane) {
  const int np = t.np;
  // slot of this lane in iteration u of row (hdr, cnt)
  auto slot = [&](unsigned long long hdr, int cnt, int u, int& s, bool& v) {
    if (SPREAD) {
      spread_slot<K>(hdr, cnt, lane, u, s, v);
    } else {
      s = lane + u * 32;
      v = s < cnt;
    }
  };
  auto pidx = [&](int kk) { return t.forward ? kk : np - 1 - kk; };
  auto row = [&](int p, int& lo, int& cnt) {
    lo = static_cast<int>(t.offs[p] - t.s0);
    cnt = static_cast<int>(t.offs[p + 1] - t.s0) - lo;
  };

  // current particle: coefficients
  int pk = pidx(0);
  int jq[K];
  double bq[K], bmq[K], cq[K];
  unsigned upm;
  bool skip;
  double diag, y;
  // next particle: raw loads
  int pk1 = np > 1 ? pidx(1) : pk, lo1, cnt1;
  row(pk1, lo1, cnt1);
  unsigned long long hdr1 = SPREAD ? t.hdr[pk1] : 0ull;
  {
    int lo, cnt;
    row(pk, lo, cnt);
    const unsigned long long hdr0 = SPREAD ? t.hdr[pk] : 0ull;
    diag = t.diag[pk];
    y = t.y[pk];
    skip = diag != diag || cnt == 0;
    upm = 0;
#pragma unroll
    for (int u = 0; u < K; ++u) {
      int s;
      bool v;
      slot(hdr0, cnt, u, s, v);
      const int jr = idle_lane_index(v ? t.nl[lo + s] : t.lbase + pk, !v, lane);  // invalid lanes: b = 0
      const int j = UNI ? (jr & 0x7fff) : jr;
      const double q = UNI ? ((v && !(jr & 0x8000)) ? t.pf[lo + s] * t.minv : 0.0) : (v ? t.qf[lo + s] : 0.0);
      const bool up = q != 0.0;                      // clamped j: never written (damping.cpp:84-86)
      jq[u] = j;
      bq[u] = v ? t.kb * t.pf[lo + s] : 0.0;
      bmq[u] = t.kb * q;
      cq[u] = -bmq[u] * (diag + bq[u]);
      if (TLSPH_CHAIN_NORATE) cq[u] *= y;
      upm |= up ? (1u << u) : 0u;
    }
    if (skip) upm = 0;
    if (TLSPH_CHAIN_NORATE) diag *= y;
  }

  for (int kk = 0; kk < np; ++kk) {
    const int li = t.lbase + pk;
    const int li1 = t.lbase + pk1;
    // (A) next particle's indices and pair factors
    int jn[K];
    double pfn[K], qfn[K];
#pragma unroll
    for (int u = 0; u < K; ++u) {
      int s;
      bool v;
      slot(hdr1, cnt1, u, s, v);
      jn[u] = idle_lane_index(v ? t.nl[lo1 + s] : li1, !v, lane);
      pfn[u] = v ? t.pf[lo1 + s] : 0.0;
      if (!UNI) qfn[u] = v ? t.qf[lo1 + s] : 0.0;
    }
    // row extents two particles ahead
    const int pk2 = kk + 2 < np ? pidx(kk + 2) : pk1;
    int lo2, cnt2;
    row(pk2, lo2, cnt2);
    const unsigned long long hdr2 = SPREAD ? t.hdr[pk2] : 0ull;

    // the chain: gathers
    double vi[D], vq[K][D];
#pragma unroll
    for (int d = 0; d < D; ++d) vi[d] = t.sv[d][li];
#pragma unroll
    for (int u = 0; u < K; ++u)
#pragma unroll
      for (int d = 0; d < D; ++d) vq[u][d] = t.sv[d][jq[u]];
    // (C) next particle's fold constants
    const double diag1 = t.diag[pk1], y1 = t.y[pk1];

    double P[D], Y[K][D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      P[d] = bq[0] * (vq[0][d] - vi[d]);
#pragma unroll
      for (int u = 1; u < K; ++u) P[d] = __fma_rn(bq[u], vq[u][d] - vi[d], P[d]);
    }
#pragma unroll
    for (int u = 0; u < K; ++u)
#pragma unroll
      for (int d = 0; d < D; ++d) Y[u][d] = TLSPH_Y(u, d);  // v_j + bm (v_j - v_i)
    if (SHUF) chain_sum<D>(P, lane);
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const double rate = TLSPH_CHAIN_NORATE ? P[d] : P[d] * y;
      if (SCATTER) {
#pragma unroll
        for (int u = 0; u < K; ++u)
          if (upm & (1u << u)) t.sv[d][jq[u]] = __fma_rn(cq[u], rate, Y[u][d]);
      }
      // i is not its own neighbour, so this store cannot race the scatter above
      if (lane == 0 && !skip) t.sv[d][li] = __fma_rn(diag, rate, vi[d]);
    }
    __syncwarp();

    // (D) next particle's coefficients
    if (UNI) {
#pragma unroll
      for (int u = 0; u < K; ++u) {
        qfn[u] = (jn[u] & 0x8000) ? 0.0 : pfn[u] * t.minv;  // invalid lanes: pfn = 0
        jn[u] &= 0x7fff;
      }
    }
    diag = diag1;
    y = y1;
    skip = diag != diag || cnt1 == 0;
    upm = 0;
#pragma unroll
    for (int u = 0; u < K; ++u) {
      const bool up = qfn[u] != 0.0;
      jq[u] = jn[u];
      bq[u] = t.kb * pfn[u];
      bmq[u] = t.kb * qfn[u];
      cq[u] = -bmq[u] * (diag + bq[u]);
      if (TLSPH_CHAIN_NORATE) cq[u] *= y;
      upm |= up ? (1u << u) : 0u;
    }
    if (skip) upm = 0;
    if (TLSPH_CHAIN_NORATE) diag *= y;
    pk = pk1;
    pk1 = pk2;
    lo1 = lo2;
    cnt1 = cnt2;
    hdr1 = hdr2;
  }
}

// The same chain with the slot block streamed from global memory (L2) instead
// of shared memory (k_sweep_fast<STREAM>): neighbour indices and pair factors
// are loaded three particles ahead, and the per-slot mass factor is formed as
// pair_factor * RN(1/m_j) from the staged stencil -- exactly the stored qf
// (state.cu k_qf), so the arithmetic is that of fast_chain. UNI (uniform
// masses): no stencil 1/m either; the factor is pair_factor * RN(1/m) unless
// bit 15 of the slot's stencil index marks a clamped j.
#ifndef TLSPH_SWEEP_STREAM_HINT
#define TLSPH_SWEEP_STREAM_HINT 0
#endif
// Measured alternatives of the streamed chain's pipeline (same-box A/B, profiles/r2c_sweep_spread.md;
// cfg4 / cfg5-weak ms per sweep, default 9.64 / 17.98):
// TLSPH_STREAM_ROTATE=0: the particle loop unrolled three times with the three raw buffers renamed
//   statically instead of moved down the pipeline every iteration (fewer instructions, but
//   10.11 / 19.05 then; the default since round 2e, see below);
// TLSPH_STREAM_U32=1: slot addresses as 32-bit indices into the body's arrays, one widening
//   multiply-add per load instead of 64-bit pointer sums (10.15 / 18.80).
// TLSPH_STREAM_ROTATE (default 0): 1 = the streamed chain's raw-load buffers are moved down the
// pipeline every iteration (18 register moves per particle); 0 = the particle loop is unrolled
// three times with the buffers renamed statically. With the shuffle-free warp sum and the folded
// rate the unrolled form wins (same-box A/B, profiles/r2e_sweep_chain_forms.md: cfg4 8.65 -> 7.90 ms
// per sweep, cfg5-weak 15.42 -> 14.60); with the round-2c chain it lost (10.11 vs 9.64).
#ifndef TLSPH_STREAM_ROTATE
#define TLSPH_STREAM_ROTATE 0
#endif
// TLSPH_STREAM_DEPTH: raw slot loads issued this many particles ahead of the particle they belong to
// (3: two whole iterations in flight, three register buffers; 2: one iteration, two buffers).
#ifndef TLSPH_STREAM_DEPTH
#define TLSPH_STREAM_DEPTH 3
#endif
#ifndef TLSPH_STREAM_U32
#define TLSPH_STREAM_U32 0
#endif
template <int K>
struct RawSlots {
  int j[K];      // stencil index (UNI: bit 15 = clamped j)
  double pf[K];  // pair factor
};

// DENSE (with UNI, SPREAD): t.nl / t.pf point at the cell's dense rows (state.cu k_dense_rows), R =
// 32 K slots per particle; lane l of iteration u owns slot 32 u + l of every row, the padding has
// pair factor 0. No row extents, group headers or load predicates.
template <int D, int K, bool UNI, bool SPREAD = false, bool DENSE = false>
__device__ __forceinline__ void fast_chain_stream(const ChainTile<D>& t, int lane) {
  const int np = t.np;
  auto pidx = [&](int kk) { return t.forward ? kk : np - 1 - kk; };
  auto pclamp = [&](int kk) { return pidx(kk < np ? kk : np - 1); };
  auto row = [&](int p, int& lo, int& cnt) {
    if (DENSE) {
      lo = p * (32 * K);
      cnt = 32 * K;
      return;
    }
    lo = static_cast<int>(t.offs[p] - t.s0);
    cnt = static_cast<int>(t.offs[p + 1] - t.s0) - lo;
  };
  // raw loads; UNI: j keeps bit 15 (clamped j) until mass_factors / coefficients strip it
  auto load_raw = [&](int lo, int cnt, unsigned long long hdr, int li, RawSlots<K>& r) {
    if (DENSE) {
#pragma unroll
      for (int u = 0; u < K; ++u) {
        r.j[u] = static_cast<int>(t.nl[lo + lane + 32 * u]);
        r.pf[u] = t.pf[lo + lane + 32 * u];
      }
      return;
    }
#pragma unroll
    for (int u = 0; u < K; ++u) {
      int s;
      bool v;
      if (SPREAD) {
        spread_slot<K>(hdr, cnt, lane, u, s, v);
      } else {
        s = lane + u * 32;
        v = s < cnt;
      }
#if TLSPH_STREAM_U32
      const unsigned g = t.s0u + static_cast<unsigned>(lo + s);
      r.j[u] = v ? static_cast<int>(t.nlb[g]) : li;
      r.pf[u] = v ? t.pfb[g] : 0.0;
#else
      // TLSPH_SWEEP_STREAM_HINT: streaming (evict-first) loads, A/B only
      r.j[u] = v ? static_cast<int>(TLSPH_SWEEP_STREAM_HINT ? __ldcs(t.nl + lo + s) : t.nl[lo + s]) : li;
      r.pf[u] = v ? (TLSPH_SWEEP_STREAM_HINT ? __ldcs(t.pf + lo + s) : t.pf[lo + s]) : 0.0;
#endif
    }
  };
  auto mass_factors = [&](const int (&j)[K], const double (&pf)[K], double (&q)[K]) {
#pragma unroll
    for (int u = 0; u < K; ++u) {
      if (UNI) {
        q[u] = (j[u] & 0x8000) ? 0.0 : pf[u] * t.minv;
      } else {
        const double my = t.smf[j[u]];
        q[u] = my > 0.0 ? pf[u] * my : 0.0;  // clamped j: never written (damping.cpp:84-86)
      }
    }
  };

  int jq[K];
  double bq[K], bmq[K], cq[K];
  unsigned upm;
  bool skip;
  double diag, y;
  auto coefficients = [&](const int (&j)[K], const double (&pf)[K], const double (&q)[K], int cnt) {
    skip = diag != diag || cnt == 0;
    upm = 0;
#pragma unroll
    for (int u = 0; u < K; ++u) {
      jq[u] = UNI ? (j[u] & 0x7fff) : j[u];
      bq[u] = t.kb * pf[u];
      bmq[u] = t.kb * q[u];
      cq[u] = -bmq[u] * (diag + bq[u]);
      if (TLSPH_CHAIN_NORATE) cq[u] *= y;
      upm |= q[u] != 0.0 ? (1u << u) : 0u;
    }
    if (skip) upm = 0;
    if (TLSPH_CHAIN_NORATE) diag *= y;
  };

  auto header = [&](int p) { return SPREAD && !DENSE ? t.hdr[p] : 0ull; };
  int pk = pidx(0);
  auto first = [&] {  // particle 0: coefficients (after the next particles' loads are in flight)
    int lo, cnt;
    RawSlots<K> r0;
    double q0[K];
    row(pk, lo, cnt);
    load_raw(lo, cnt, header(pk), t.lbase + pk, r0);
#pragma unroll
    for (int u = 0; u < K; ++u) r0.j[u] = idle_lane_index(r0.j[u], r0.pf[u] == 0.0, lane);
    diag = t.diag[pk];
    y = t.y[pk];
    mass_factors(r0.j, r0.pf, q0);
    coefficients(r0.j, r0.pf, q0, cnt);
  };
  int pk1 = pclamp(1);

  // One particle of the chain (pk); `use` holds the raw slots of the next one (pk1, cnt_next slots),
  // whose coefficients are formed after the scatter.
  auto update = [&](RawSlots<K>& use, int cnt_next) {
    const int li = t.lbase + pk;
    // the next particle's idle lanes (pair factor 0: no slot, or a slot that contributes nothing)
#pragma unroll
    for (int u = 0; u < K; ++u) use.j[u] = idle_lane_index(use.j[u], use.pf[u] == 0.0, lane);
    // the chain: gathers
    double vi[D], vq[K][D];
#pragma unroll
    for (int d = 0; d < D; ++d) vi[d] = t.sv[d][li];
#pragma unroll
    for (int u = 0; u < K; ++u)
#pragma unroll
      for (int d = 0; d < D; ++d) vq[u][d] = t.sv[d][jq[u]];
    const double diag1 = t.diag[pk1], y1 = t.y[pk1];

    double P[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      P[d] = bq[0] * (vq[0][d] - vi[d]);
#pragma unroll
      for (int u = 1; u < K; ++u) P[d] = __fma_rn(bq[u], vq[u][d] - vi[d], P[d]);
    }
#if !TLSPH_Y_LATE
    double Y[K][D];
#pragma unroll
    for (int u = 0; u < K; ++u)
#pragma unroll
      for (int d = 0; d < D; ++d) Y[u][d] = TLSPH_Y(u, d);  // v_j + bm (v_j - v_i)
#endif
    chain_sum<D>(P, lane);
    double qfn[K];
    mass_factors(use.j, use.pf, qfn);  // the next particle
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const double rate = TLSPH_CHAIN_NORATE ? P[d] : P[d] * y;
#pragma unroll
      for (int u = 0; u < K; ++u)
#if TLSPH_Y_LATE
        if (upm & (1u << u)) t.sv[d][jq[u]] = __fma_rn(cq[u], rate, TLSPH_Y(u, d));
#else
        if (upm & (1u << u)) t.sv[d][jq[u]] = __fma_rn(cq[u], rate, Y[u][d]);
#endif
      // i is not its own neighbour, so this store cannot race the scatter above
      if (lane == 0 && !skip) t.sv[d][li] = __fma_rn(diag, rate, vi[d]);
    }
    __syncwarp();

    diag = diag1;
    y = y1;
    coefficients(use.j, use.pf, qfn, cnt_next);
  };

#if TLSPH_STREAM_DEPTH == 2
  // Raw loads one particle ahead of their use: particle 1 in flight; particle 2: row extents.
  int pk2 = pclamp(2);
  int lo1, cnt1, lo2, cnt2;
  RawSlots<K> ra, rb;
  row(pk1, lo1, cnt1);
  row(pk2, lo2, cnt2);
  unsigned long long hdr2 = header(pk2);
  load_raw(lo1, cnt1, header(pk1), t.lbase + pk1, ra);
  first();
  // `use` holds particle kk+1's raw slots (loaded one iteration ago), `fill` receives particle kk+2's
  auto step = [&](int kk, RawSlots<K>& use, RawSlots<K>& fill) {
    load_raw(lo2, cnt2, hdr2, t.lbase + pk2, fill);
    const int pk3 = pclamp(kk + 3);
    int lo3, cnt3;
    row(pk3, lo3, cnt3);
    hdr2 = header(pk3);
    update(use, cnt1);
    pk = pk1;
    pk1 = pk2;
    pk2 = pk3;
    cnt1 = cnt2;
    lo2 = lo3;
    cnt2 = cnt3;
  };
#if TLSPH_STREAM_ROTATE
  for (int kk = 0; kk < np; ++kk) {
    step(kk, ra, rb);
#pragma unroll
    for (int u = 0; u < K; ++u) {
      ra.j[u] = rb.j[u];
      ra.pf[u] = rb.pf[u];
    }
  }
#else
  for (int kk = 0;;) {
    step(kk, ra, rb);
    if (++kk >= np) break;
    step(kk, rb, ra);
    if (++kk >= np) break;
  }
#endif
#else
  // Raw loads two particles ahead of their use: particles 1, 2 in flight; particle 3: row extents.
  int pk2 = pclamp(2), pk3 = pclamp(3);
  int lo1, cnt1, lo2, cnt2, lo3, cnt3;
  RawSlots<K> ra, rb, rc;
  row(pk1, lo1, cnt1);
  row(pk2, lo2, cnt2);
  row(pk3, lo3, cnt3);
  unsigned long long hdr3 = header(pk3);
  load_raw(lo1, cnt1, header(pk1), t.lbase + pk1, ra);
  load_raw(lo2, cnt2, header(pk2), t.lbase + pk2, rb);
  first();
  // `use` holds particle kk+1's raw slots (loaded two iterations ago), `fill` receives particle kk+3's
  auto step = [&](int kk, RawSlots<K>& use, RawSlots<K>& fill) {
    load_raw(lo3, cnt3, hdr3, t.lbase + pk3, fill);
    const int pk4 = pclamp(kk + 4);
    int lo4, cnt4;
    row(pk4, lo4, cnt4);
    hdr3 = header(pk4);
    update(use, cnt1);
    pk = pk1;
    pk1 = pk2;
    pk2 = pk3;
    pk3 = pk4;
    cnt1 = cnt2;
    cnt2 = cnt3;
    lo3 = lo4;
    cnt3 = cnt4;
  };
#if TLSPH_STREAM_ROTATE
  for (int kk = 0; kk < np; ++kk) {
    step(kk, ra, rc);
#pragma unroll
    for (int u = 0; u < K; ++u) {
      ra.j[u] = rb.j[u];
      ra.pf[u] = rb.pf[u];
      rb.j[u] = rc.j[u];
      rb.pf[u] = rc.pf[u];
    }
  }
#else
  for (int kk = 0;;) {
    step(kk, ra, rc);
    if (++kk >= np) break;
    step(kk, rb, ra);
    if (++kk >= np) break;
    step(kk, rc, rb);
    if (++kk >= np) break;
  }
#endif
#endif
}

}  // namespace tlsph_cuda
