// Ablation microbenchmark of the damping sweep's per-particle chain (one warp,
// shared-memory stencil, K slots per lane), to attribute the cycles per
// particle to loads / shuffle reduction / scatter stores.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int S = 512, NP = 17, K = 3, D = 3, CNT = 76;

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

template <int MODE>  // 0 full, 1 no scatter stores, 2 no shuffles, 3 no syncwarp/lane0 store, 4 loads+partials only
__global__ void chain(const int* nloc, const double* b_in, double* out, long long* cyc, int reps) {
  __shared__ double sv[D][S];
  __shared__ int snl[NP * CNT];
  __shared__ double sb[NP * CNT];
  for (int e = threadIdx.x; e < S; e += 32)
    for (int d = 0; d < D; ++d) sv[d][e] = 0.001 * e + d;
  for (int e = threadIdx.x; e < NP * CNT; e += 32) {
    snl[e] = nloc[e];
    sb[e] = b_in[e];
  }
  __syncwarp();
  const int lane = threadIdx.x;
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    for (int kk = 0; kk < NP; ++kk) {
      const int li = 200 + kk;
      const int lo = kk * CNT;
      int jq[K];
      double bq[K];
#pragma unroll
      for (int u = 0; u < K; ++u) {
        const int s = lane + 32 * u;
        const bool v = s < CNT;
        jq[u] = v ? snl[lo + s] : li;
        bq[u] = v ? sb[lo + s] : 0.0;
      }
      double vi[D], vq[K][D], R[D];
#pragma unroll
      for (int d = 0; d < D; ++d) vi[d] = sv[d][li];
#pragma unroll
      for (int u = 0; u < K; ++u)
#pragma unroll
        for (int d = 0; d < D; ++d) vq[u][d] = sv[d][jq[u]];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        double r = 0.0;
#pragma unroll
        for (int u = 0; u < K; ++u) r = r - bq[u] * (vi[d] - vq[u][d]);
        R[d] = (MODE == 2 || MODE == 4) ? r : warp_sum(r);
      }
      double vnew[D], rate[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        rate[d] = R[d] * 1e-3;
        vnew[d] = vi[d] + 0.5 * rate[d];
      }
      if (MODE != 1 && MODE != 4) {
#pragma unroll
        for (int u = 0; u < K; ++u)
#pragma unroll
          for (int d = 0; d < D; ++d) {
            const double pred = vq[u][d] - bq[u] * rate[d];
            if (lane + 32 * u < CNT) sv[d][jq[u]] = vq[u][d] - 0.3 * (vnew[d] - pred);
          }
      }
      if (MODE != 3 && MODE != 4) {
        if (lane == 0)
#pragma unroll
          for (int d = 0; d < D; ++d) sv[d][li] = vnew[d];
        __syncwarp();
      } else {
#pragma unroll
        for (int d = 0; d < D; ++d) sv[d][li] = vnew[d];
      }
    }
  }
  long long t1 = clock64();
  if (lane == 0) {
    cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x] = sv[0][0] + sv[1][1];
  }
}


// component-split chain: lanes [8d, 8d+8) own component d, KC slots per lane
template <int MODE>
__global__ void chain_split(const int* nloc, const double* b_in, double* out, long long* cyc, int reps) {
  __shared__ double sv[D][S];
  __shared__ int snl[NP * CNT];
  __shared__ double sb[NP * CNT];
  for (int e = threadIdx.x; e < S; e += 32)
    for (int d = 0; d < D; ++d) sv[d][e] = 0.001 * e + d;
  for (int e = threadIdx.x; e < NP * CNT; e += 32) {
    snl[e] = nloc[e];
    sb[e] = b_in[e];
  }
  __syncwarp();
  constexpr int G = 8, KC = (CNT + G - 1) / G;
  const int lane = threadIdx.x, grp = lane / G, gl = lane % G;
  const int dcomp = grp < D ? grp : 0;
  double* vd = sv[dcomp];
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    for (int kk = 0; kk < NP; ++kk) {
      const int li = 200 + kk;
      const int lo = kk * CNT;
      int jq[KC];
      double bq[KC], vq[KC];
#pragma unroll
      for (int u = 0; u < KC; ++u) {
        const int s = gl + G * u;
        const bool v = s < CNT;
        jq[u] = v ? snl[lo + s] : li;
        bq[u] = v ? sb[lo + s] : 0.0;
      }
      const double vi = vd[li];
#pragma unroll
      for (int u = 0; u < KC; ++u) vq[u] = vd[jq[u]];
      double p[KC];
#pragma unroll
      for (int u = 0; u < KC; ++u) p[u] = bq[u] * (vi - vq[u]);
      // pairwise tree of the lane's partials
#pragma unroll
      for (int w = 1; w < KC; w <<= 1)
#pragma unroll
        for (int u = 0; u + w < KC; u += 2 * w) p[u] = p[u] + p[u + w];
      double r = -p[0];
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
      const double rate = r * 1e-3;
      const double vnew = vi + 0.5 * rate;
#pragma unroll
      for (int u = 0; u < KC; ++u) {
        double nv;
        if (MODE == 0) {
          const double pred = vq[u] - bq[u] * rate;
          nv = vq[u] - 0.3 * (vnew - pred);
        } else {
          nv = __fma_rn(1.3, vq[u], -(0.3 * vnew + 0.3 * bq[u] * rate));
        }
        if (grp < D && gl + G * u < CNT) vd[jq[u]] = nv;
      }
      if (gl == 0 && grp < D) vd[li] = vnew;
      __syncwarp();
    }
  }
  long long t1 = clock64();
  if (lane == 0) {
    cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x] = sv[0][0] + sv[1][1];
  }
}

int main() {
  int h_nl[NP * CNT];
  double h_b[NP * CNT];
  srand(1);
  for (int k = 0; k < NP; ++k) {
    // distinct neighbours per row, none equal to the row's own index
    int used[S] = {0};
    used[200 + k] = 1;
    for (int s = 0; s < CNT; ++s) {
      int j;
      do j = rand() % S; while (used[j]);
      used[j] = 1;
      h_nl[k * CNT + s] = j;
      h_b[k * CNT + s] = -1e-3 * (1 + rand() % 100);
    }
  }
  int* nl;
  double *b, *out;
  long long* cyc;
  cudaMalloc(&nl, sizeof(h_nl));
  cudaMalloc(&b, sizeof(h_b));
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMalloc(&cyc, 1024 * sizeof(long long));
  cudaMemcpy(nl, h_nl, sizeof(h_nl), cudaMemcpyHostToDevice);
  cudaMemcpy(b, h_b, sizeof(h_b), cudaMemcpyHostToDevice);
  const char* names[] = {"full", "no scatter", "no shuffles", "no lane0+syncwarp", "loads+partials only"};
  for (int blocks : {1, 148 * 4}) {
    for (int mode = 0; mode < 5; ++mode) {
      const int reps = 50;
      for (int w = 0; w < 2; ++w) {
        switch (mode) {
          case 0: chain<0><<<blocks, 32>>>(nl, b, out, cyc, reps); break;
          case 1: chain<1><<<blocks, 32>>>(nl, b, out, cyc, reps); break;
          case 2: chain<2><<<blocks, 32>>>(nl, b, out, cyc, reps); break;
          case 3: chain<3><<<blocks, 32>>>(nl, b, out, cyc, reps); break;
          case 4: chain<4><<<blocks, 32>>>(nl, b, out, cyc, reps); break;
        }
      }
      long long c = 0;
      cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
      printf("blocks %4d %-22s %8.1f cycles/particle\n", blocks, names[mode], double(c) / (reps * NP));
    }
  }
  for (int blocks : {1, 148 * 4}) {
    for (int mode = 0; mode < 2; ++mode) {
      const int reps = 50;
      for (int w = 0; w < 2; ++w) {
        if (mode == 0) chain_split<0><<<blocks, 32>>>(nl, b, out, cyc, reps);
        else chain_split<1><<<blocks, 32>>>(nl, b, out, cyc, reps);
      }
      long long c = 0;
      cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
      printf("blocks %4d split %-16s %8.1f cycles/particle\n", blocks, mode ? "fma-scatter" : "exact-scatter",
             double(c) / (reps * NP));
    }
  }
  return 0;
}
