// Colour-scheduled, operator-split implicit viscous damping sweep.
//
// Reference: proj/src/tlsph/damping.cpp:53-182 (particle_split_update,
// pairwise_split_update, strang_damping_sweep), neighbors.cpp:143-174
// (block_sweep), neighbors.cpp:61-77 (3^D residue colouring).
//
// One launch per colour phase: colour b holds the cells whose coordinates
// are congruent to b's residues mod 3 on every axis; their 3^D stencils are
// disjoint (neighbors.hpp:50-52), so each cell is one independent task. One
// warp owns one cell:
//   1. stage the cell's stencil (3^(D-1) contiguous x-rows of the cell-sorted
//      arrays) of v, m and the clamp flag into shared memory;
//   2. run the cell's particles in order (ascending id forward, descending on
//      the reverse leg, damping.cpp:112-121); for particle i the lanes split
//      its CSR slots, reduce residual / sum b / sum b^2 with warp shuffles
//      (FAST) or lane 0 folds them in slot order (ORDERED, bit-exact), then
//      apply the momentum-conserving neighbour correction lane-parallel;
//   3. write the stencil back (same-colour stencils are disjoint: no races).
// The pairwise scheme runs the same staging with lane 0 applying the 2x2
// pair solves in the palindromic slot order (damping.cpp:161-176).
#include <algorithm>
#include <cmath>

#include "system.cuh"

namespace tlsph_cuda {

namespace {

unsigned grid_for(long long n, int block) { return static_cast<unsigned>((n + block - 1) / block); }

constexpr int kSweepWarps = 4;

struct Phase {
  int res[3];     // colour residues per axis
  int cnt[3];     // cells of this colour per axis
  long long ncol; // cells in the colour
  int forward;
  int stride;     // staged stencil capacity per warp (elements)
  double eta;
  double dt;      // used when dt_from_scalars == 0
  int dt_from_scalars;
};

template <int D>
__host__ __device__ constexpr int colour_count() { return D == 2 ? 9 : 27; }

// bytes of staged state per warp
template <int D>
__host__ __device__ size_t warp_smem_bytes(int stride) {
  return static_cast<size_t>(stride) * (sizeof(double) * (D + 1) + 1);
}

template <int D, int SCHEME, bool ORDERED>
__global__ void __launch_bounds__(kSweepWarps * kWarp)
k_sweep_phase(DFields f, Phase ph, const DScalars* __restrict__ sc) {
  if (ph.dt_from_scalars && sc->halt) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const long long k = static_cast<long long>(blockIdx.x) * kSweepWarps + warp;
  if (k >= ph.ncol) return;
  // cell coordinates of task k in colour (res)
  int c[3];
  c[0] = ph.res[0] + 3 * static_cast<int>(k % ph.cnt[0]);
  c[1] = ph.res[1] + 3 * static_cast<int>((k / ph.cnt[0]) % ph.cnt[1]);
  c[2] = D == 3 ? ph.res[2] + 3 * static_cast<int>(k / (static_cast<long long>(ph.cnt[0]) * ph.cnt[1])) : 0;
  const long long lin = cell_linear<D>(c, f.dims);
  const long long p0 = f.cell_start[lin], p1 = f.cell_start[lin + 1];
  if (p0 == p1) return;

  const int S = ph.stride;
  unsigned char* wbase = smem + static_cast<size_t>(warp) * warp_smem_bytes<D>(S);
  double* sv[D];
#pragma unroll
  for (int d = 0; d < D; ++d) sv[d] = reinterpret_cast<double*>(wbase) + d * S;
  double* sm = reinterpret_cast<double*>(wbase) + D * S;
  uint8_t* sf = wbase + sizeof(double) * (D + 1) * S;

  Stencil<D> st;
  stencil_segments<D>(f.cell_start, f.dims, c, st);
#pragma unroll
  for (int q = 0; q < Stencil<D>::kSegs; ++q) {
    const long long g0 = st.start[q];
    const int b = st.base[q];
    for (int e = lane; e < st.len[q]; e += kWarp) {
#pragma unroll
      for (int d = 0; d < D; ++d) sv[d][b + e] = f.v[d][g0 + e];
      sm[b + e] = f.m[g0 + e];
      sf[b + e] = f.flag[g0 + e];
    }
  }
  __syncwarp();

  const double dt = ph.dt_from_scalars ? sc->dt : ph.dt;
  const double dt_half = 0.5 * dt;
  const double eta = ph.eta;
  const int center = D == 2 ? 1 : 4;
  const long long cbase = st.start[center];
  const int lbase = st.base[center];
  const long long np = p1 - p0;

  for (long long kk = 0; kk < np; ++kk) {
    const long long i = ph.forward ? p0 + kk : p1 - 1 - kk;
    const int li = lbase + static_cast<int>(i - cbase);
    if (sf[li]) continue;  // constrained i is skipped (damping.cpp:151,163)
    const long long lo = f.offs[i], hi = f.offs[i + 1];
    if (SCHEME == TLSPH_SCHEME_PARTICLE_SPLIT) {
      if (lo == hi) continue;
      double vi[D];
#pragma unroll
      for (int d = 0; d < D; ++d) vi[d] = sv[d][li];
      double R[D], sb = 0.0, sb2 = 0.0;
#pragma unroll
      for (int d = 0; d < D; ++d) R[d] = 0.0;
      if (ORDERED) {
        if (lane == 0) {
          for (long long s = lo; s < hi; ++s) {
            const double b = eta * f.pf[s] * dt_half;
            const int j = f.nloc[s];
#pragma unroll
            for (int d = 0; d < D; ++d) R[d] = R[d] - b * (vi[d] - sv[d][j]);
            sb = sb + b;
            sb2 = sb2 + b * b;
          }
        }
#pragma unroll
        for (int d = 0; d < D; ++d) R[d] = __shfl_sync(0xffffffffu, R[d], 0);
        sb = __shfl_sync(0xffffffffu, sb, 0);
        sb2 = __shfl_sync(0xffffffffu, sb2, 0);
      } else {
        for (long long s = lo + lane; s < hi; s += kWarp) {
          const double b = eta * f.pf[s] * dt_half;
          const int j = f.nloc[s];
#pragma unroll
          for (int d = 0; d < D; ++d) R[d] = R[d] - b * (vi[d] - sv[d][j]);
          sb = sb + b;
          sb2 = sb2 + b * b;
        }
#pragma unroll
        for (int d = 0; d < D; ++d) R[d] = warp_sum(R[d]);
        sb = warp_sum(sb);
        sb2 = warp_sum(sb2);
      }
      const double diag = sb - sm[li];
      const double denom = diag * diag + sb2;
      double rate[D], vnew[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        rate[d] = R[d] / denom;
        vnew[d] = vi[d] + diag * rate[d];
      }
      // neighbour correction: every j is distinct within the row, so the
      // lane-parallel order is bit-identical to the reference loop.
      for (long long s = lo + lane; s < hi; s += kWarp) {
        const double b = eta * f.pf[s] * dt_half;
        const int j = f.nloc[s];
        if (!sf[j]) {
          const double bm = b / sm[j];
#pragma unroll
          for (int d = 0; d < D; ++d) {
            const double vj = sv[d][j];
            const double pred = vj - b * rate[d];
            sv[d][j] = vj - bm * (vnew[d] - pred);
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int d = 0; d < D; ++d) sv[d][li] = vnew[d];
      }
      __syncwarp();
    } else {
      // pairwise split: palindromic chain of 2x2 solves at dt/4 (damping.cpp:161-176)
      if (lane == 0) {
        const double dt_pair = 0.5 * dt_half;
        const double mi = sm[li];
        double vi[D];
#pragma unroll
        for (int d = 0; d < D; ++d) vi[d] = sv[d][li];
        for (int pass = 0; pass < 2; ++pass) {
          const long long cnt = hi - lo;
          for (long long t = 0; t < cnt; ++t) {
            const long long s = pass == 0 ? lo + t : hi - 1 - t;
            const double b = eta * f.pf[s] * dt_pair;
            const int j = f.nloc[s];
            const double mj = sm[j];
            const double denom = mi * mj - (mi + mj) * b;
            const double kf = b / denom;
            const bool upd = !sf[j];
#pragma unroll
            for (int d = 0; d < D; ++d) {
              const double vj = sv[d][j];
              const double scaled = kf * (vi[d] - vj);
              vi[d] = vi[d] + mj * scaled;
              if (upd) sv[d][j] = vj - mi * scaled;
            }
          }
        }
#pragma unroll
        for (int d = 0; d < D; ++d) sv[d][li] = vi[d];
      }
      __syncwarp();
    }
  }

  // write the stencil back
#pragma unroll
  for (int q = 0; q < Stencil<D>::kSegs; ++q) {
    const long long g0 = st.start[q];
    const int b = st.base[q];
    for (int e = lane; e < st.len[q]; e += kWarp) {
#pragma unroll
      for (int d = 0; d < D; ++d) f.v[d][g0 + e] = sv[d][b + e];
    }
  }
}

// ------------------------------------------------------------------ single-particle operators
template <int D>
__global__ void k_particle_split_one(DFields f, long long i, double eta, double dt_half) {
  if (threadIdx.x != 0) return;
  const long long lo = f.offs[i], hi = f.offs[i + 1];
  if (lo == hi) return;
  double vi[D], R[D], sb = 0.0, sb2 = 0.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    vi[d] = f.v[d][i];
    R[d] = 0.0;
  }
  for (long long s = lo; s < hi; ++s) {
    const int j = f.nbr[s];
    const double b = eta * f.pf[s] * dt_half;
#pragma unroll
    for (int d = 0; d < D; ++d) R[d] = R[d] - b * (vi[d] - f.v[d][j]);
    sb = sb + b;
    sb2 = sb2 + b * b;
  }
  const double diag = sb - f.m[i];
  const double denom = diag * diag + sb2;
  double rate[D], vnew[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    rate[d] = R[d] / denom;
    vnew[d] = vi[d] + diag * rate[d];
  }
  for (long long s = lo; s < hi; ++s) {
    const int j = f.nbr[s];
    const double b = eta * f.pf[s] * dt_half;
    if (!f.flag[j]) {
      const double bm = b / f.m[j];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const double vj = f.v[d][j];
        const double pred = vj - b * rate[d];
        f.v[d][j] = vj - bm * (vnew[d] - pred);
      }
    }
  }
#pragma unroll
  for (int d = 0; d < D; ++d) f.v[d][i] = vnew[d];
}

template <int D>
__global__ void k_pairwise_one(DFields f, long long i, long long s, double eta, double dt_half) {
  if (threadIdx.x != 0) return;
  const int j = f.nbr[s];
  const double b = eta * f.pf[s] * dt_half;
  const double mi = f.m[i], mj = f.m[j];
  const double denom = mi * mj - (mi + mj) * b;
  const double kf = b / denom;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double vi = f.v[d][i], vj = f.v[d][j];
    const double scaled = kf * (vi - vj);
    f.v[d][i] = vi + mj * scaled;
    if (!f.flag[j]) f.v[d][j] = vj - mi * scaled;
  }
}

// explicit_damping_accel (damping.cpp:36-51): out_i = (eta/m_i) sum G_ij v_ij
template <int D>
__global__ void k_explicit_accel(DFields f, double eta, double* __restrict__ out /* SoA D x n */) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= f.n) return;
  double acc[D], vi[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    acc[d] = 0.0;
    vi[d] = f.v[d][i];
  }
  for (long long s = f.offs[i]; s < f.offs[i + 1]; ++s) {
    const int j = f.nbr[s];
    const double g = f.pf[s];
#pragma unroll
    for (int d = 0; d < D; ++d) acc[d] = acc[d] + g * (vi[d] - f.v[d][j]);
  }
  const double k = eta / f.m[i];
#pragma unroll
  for (int d = 0; d < D; ++d) out[d * f.n + i] = k * acc[d];
}

// runner.cpp:363-367: v += dt * a_visc, then constraints.
template <int D>
__global__ void k_explicit_update(DFields f, const double* __restrict__ acc, const DScalars* sc, double dt_fixed,
                                  int dt_from_scalars) {
  if (dt_from_scalars && sc->halt) return;
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= f.n) return;
  const double dt = dt_from_scalars ? sc->dt : dt_fixed;
#pragma unroll
  for (int d = 0; d < D; ++d) f.v[d][i] = f.flag[i] ? 0.0 : f.v[d][i] + dt * acc[d * f.n + i];
}

template <int D>
__global__ void k_explicit_accel_loop(DFields f, double eta, double* __restrict__ out, const DScalars* sc) {
  if (sc->halt) return;
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= f.n) return;
  double acc[D], vi[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    acc[d] = 0.0;
    vi[d] = f.v[d][i];
  }
  for (long long s = f.offs[i]; s < f.offs[i + 1]; ++s) {
    const int j = f.nbr[s];
    const double g = f.pf[s];
#pragma unroll
    for (int d = 0; d < D; ++d) acc[d] = acc[d] + g * (vi[d] - f.v[d][j]);
  }
  const double k = eta / f.m[i];
#pragma unroll
  for (int d = 0; d < D; ++d) out[d * f.n + i] = k * acc[d];
}

template <int D, int SCHEME, bool ORDERED>
void launch_phase(const DevSystem& s, const DFields& f, const Phase& ph) {
  const size_t smem = kSweepWarps * warp_smem_bytes<D>(ph.stride);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    CK(cudaFuncSetAttribute(k_sweep_phase<D, SCHEME, ORDERED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(smem)));
    configured = smem;
  }
  k_sweep_phase<D, SCHEME, ORDERED><<<grid_for(ph.ncol, kSweepWarps), kSweepWarps * kWarp, smem, s.stream>>>(
      f, ph, s.scal.p);
}

template <int D>
void enqueue_sweep_d(DevSystem& s, int scheme, double eta, double dt, bool from_scal) {
  if (!s.stencil_ok)
    throw DevError(TLSPH_ERR_INVALID_ARGUMENT,
                   "damping sweep needs every neighbour inside the 3^D cell stencil (neighbors.hpp:50-52)");
  const DFields f = s.fields();
  Phase ph{};
  ph.eta = eta;
  ph.dt = dt;
  ph.dt_from_scalars = from_scal ? 1 : 0;
  ph.stride = (std::max(s.max_stencil, 1) + 7) & ~7;  // keeps every staged array 8-byte aligned
  const bool ord = s.reduction == TLSPH_REDUCTION_ORDERED;
  constexpr int nb = colour_count<D>();
  for (int pass = 0; pass < 2; ++pass) {
    ph.forward = pass == 0;
    for (int bb = 0; bb < nb; ++bb) {
      const int b = pass == 0 ? bb : nb - 1 - bb;
      int rem = b;
      long long total = 1;
      for (int d = 0; d < 3; ++d) {
        if (d < D) {
          ph.res[d] = rem % 3;
          rem /= 3;
          ph.cnt[d] = s.dims[d] > ph.res[d] ? (s.dims[d] - ph.res[d] + 2) / 3 : 0;
        } else {
          ph.res[d] = 0;
          ph.cnt[d] = 1;
        }
        total *= ph.cnt[d];
      }
      ph.ncol = total;
      if (total == 0) continue;  // empty colour (neighbors.cpp:152)
      if (scheme == TLSPH_SCHEME_PARTICLE_SPLIT) {
        if (ord) launch_phase<D, TLSPH_SCHEME_PARTICLE_SPLIT, true>(s, f, ph);
        else launch_phase<D, TLSPH_SCHEME_PARTICLE_SPLIT, false>(s, f, ph);
      } else {
        launch_phase<D, TLSPH_SCHEME_PAIRWISE_SPLIT, false>(s, f, ph);
      }
    }
  }
  CK_LAUNCH("k_sweep_phase");
}

}  // namespace

void DevSystem::enqueue_sweep(int scheme, double eta_tilde, double dt_fixed, bool dt_from_scalars) {
  if (D == 2) enqueue_sweep_d<2>(*this, scheme, eta_tilde, dt_fixed, dt_from_scalars);
  else enqueue_sweep_d<3>(*this, scheme, eta_tilde, dt_fixed, dt_from_scalars);
}

void DevSystem::damping_sweep(int scheme, double eta_tilde, double dt, int count) {
  if (eta_tilde == 0.0) return;  // damping.cpp:132
  if (scheme == TLSPH_SCHEME_EXPLICIT)
    throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "the explicit scheme is integrated directly, not swept");
  if (scheme != TLSPH_SCHEME_PARTICLE_SPLIT && scheme != TLSPH_SCHEME_PAIRWISE_SPLIT)
    throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "unknown damping scheme");
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, stream));
  for (int c = 0; c < count; ++c) enqueue_sweep(scheme, eta_tilde, dt, false);
  CK(cudaEventRecord(e1, stream));
  CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  last_elapsed = ms * 1e-3;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

void DevSystem::particle_split_update(long long i, double eta, double dt_half) {
  if (i < 0 || i >= n) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "particle index out of range");
  int si = 0;
  CK(cudaMemcpy(&si, rank.p + i, sizeof(int), cudaMemcpyDeviceToHost));
  DFields f = fields();
  if (D == 2) k_particle_split_one<2><<<1, 32, 0, stream>>>(f, si, eta, dt_half);
  else k_particle_split_one<3><<<1, 32, 0, stream>>>(f, si, eta, dt_half);
  CK_LAUNCH("k_particle_split_one");
  sync();
}

void DevSystem::pairwise_split_update(long long i, long long slot, double eta, double dt_half) {
  if (i < 0 || i >= n) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "particle index out of range");
  int si = 0;
  CK(cudaMemcpy(&si, rank.p + i, sizeof(int), cudaMemcpyDeviceToHost));
  // `slot` is a reference-order CSR slot. Sorted rows keep the reference slot
  // order, so the offset within row i carries over; the reference row start
  // comes from a host prefix sum of the row sizes.
  std::vector<long long> ro(2);
  CK(cudaMemcpy(ro.data(), offs.p + si, 2 * sizeof(long long), cudaMemcpyDeviceToHost));
  std::vector<long long> hoff(static_cast<size_t>(n + 1));
  {
    std::vector<long long> so(static_cast<size_t>(n + 1));
    std::vector<int> hperm(static_cast<size_t>(n));
    CK(cudaMemcpy(so.data(), offs.p, (n + 1) * sizeof(long long), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hperm.data(), perm.p, n * sizeof(int), cudaMemcpyDeviceToHost));
    std::vector<long long> rc(static_cast<size_t>(n));
    for (long long s = 0; s < n; ++s) rc[hperm[s]] = so[s + 1] - so[s];
    hoff[0] = 0;
    for (long long r = 0; r < n; ++r) hoff[r + 1] = hoff[r] + rc[r];
  }
  const long long within = slot - hoff[i];
  if (within < 0 || within >= ro[1] - ro[0]) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "slot out of row range");
  DFields f = fields();
  if (D == 2) k_pairwise_one<2><<<1, 32, 0, stream>>>(f, si, ro[0] + within, eta, dt_half);
  else k_pairwise_one<3><<<1, 32, 0, stream>>>(f, si, ro[0] + within, eta, dt_half);
  CK_LAUNCH("k_pairwise_one");
  sync();
}

void DevSystem::explicit_damping_accel(double eta, double* out_host) {
  DBuf<double> acc, aos;
  acc.alloc(static_cast<size_t>(n) * D);
  DFields f = fields();
  if (D == 2) k_explicit_accel<2><<<grid_for(n, 128), 128, 0, stream>>>(f, eta, acc.p);
  else k_explicit_accel<3><<<grid_for(n, 128), 128, 0, stream>>>(f, eta, acc.p);
  CK_LAUNCH("k_explicit_accel");
  std::vector<double> soa(static_cast<size_t>(n) * D);
  std::vector<int> hperm(static_cast<size_t>(n));
  CK(cudaMemcpyAsync(soa.data(), acc.p, soa.size() * sizeof(double), cudaMemcpyDeviceToHost, stream));
  CK(cudaMemcpyAsync(hperm.data(), perm.p, n * sizeof(int), cudaMemcpyDeviceToHost, stream));
  sync();
  for (long long s = 0; s < n; ++s)
    for (int d = 0; d < D; ++d) out_host[static_cast<long long>(hperm[s]) * D + d] = soa[d * n + s];
}

// loop helpers for explicit damping (loop.cu)
void enqueue_explicit(DevSystem& s, double eta, double* acc) {
  DFields f = s.fields();
  if (s.D == 2) {
    k_explicit_accel_loop<2><<<grid_for(s.n, 128), 128, 0, s.stream>>>(f, eta, acc, s.scal.p);
    k_explicit_update<2><<<grid_for(s.n, 256), 256, 0, s.stream>>>(f, acc, s.scal.p, 0.0, 1);
  } else {
    k_explicit_accel_loop<3><<<grid_for(s.n, 128), 128, 0, s.stream>>>(f, eta, acc, s.scal.p);
    k_explicit_update<3><<<grid_for(s.n, 256), 256, 0, s.stream>>>(f, acc, s.scal.p, 0.0, 1);
  }
  CK_LAUNCH("explicit damping");
}

}  // namespace tlsph_cuda
