// Single-particle damping operators, the explicit scheme and the host side
// of strang_damping_sweep. The colour-phase sweep kernel is in sweep.cu.
//
// Reference: proj/src/tlsph/damping.cpp:36-182.
#include <algorithm>
#include <cmath>

#include "system.cuh"

namespace tlsph_cuda {

namespace {

unsigned grid_for(long long n, int block) { return static_cast<unsigned>((n + block - 1) / block); }

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

}  // namespace

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
