// Cycle-stamped single-component chain (one warp), to attribute the
// per-particle latency of fast_chain_comp to its stages on this B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/chain_probe tools/chain_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int S = 512, NP = 18, K = 3, CNT = 76;

__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
  return c;
}

__global__ void probe(const uint16_t* nloc, const double* pf, long long* out) {
  __shared__ double sv[S];
  __shared__ double sb[NP * CNT];
  __shared__ uint16_t snl[NP * CNT];
  const int lane = threadIdx.x;
  for (int e = lane; e < S; e += 32) sv[e] = 0.001 * e;
  for (int e = lane; e < NP * CNT; e += 32) {
    snl[e] = nloc[e];
    sb[e] = pf[e];
  }
  __syncwarp();
  long long acc[8] = {0};
  for (int rep = 0; rep < 20; ++rep) {
    for (int kk = 0; kk < NP; ++kk) {
      const int li = 200 + kk;
      int jq[K];
      double bq[K];
#pragma unroll
      for (int u = 0; u < K; ++u) {
        const int s = lane + 32 * u;
        const bool v = s < CNT;
        jq[u] = v ? snl[kk * CNT + s] : li;
        bq[u] = v ? sb[kk * CNT + s] : 0.0;
      }
      // make the metadata ready before timing starts
      double dep = 0.0;
#pragma unroll
      for (int u = 0; u < K; ++u) dep += bq[u] + jq[u];
      if (dep == 12345.0) sv[0] = dep;
      __syncwarp();
      const long long t0 = clk();
      const double vi = sv[li];
      double vq[K];
#pragma unroll
      for (int u = 0; u < K; ++u) vq[u] = sv[jq[u]];
      double w[K];
#pragma unroll
      for (int u = 0; u < K; ++u) w[u] = vq[u] - vi;
      const long long t1 = clk();
      double P = bq[0] * w[0];
#pragma unroll
      for (int u = 1; u < K; ++u) P = __fma_rn(bq[u], w[u], P);
      double Y[K];
#pragma unroll
      for (int u = 0; u < K; ++u) Y[u] = __fma_rn(0.3, w[u], vq[u]);
      const double Pl = P;
      const long long t2 = clk();
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) P += __shfl_xor_sync(0xffffffffu, P, o);
      const long long t3 = clk();
      const double rate = P * 0.5;
#pragma unroll
      for (int u = 0; u < K; ++u)
        if (lane + 32 * u < CNT) sv[jq[u]] = __fma_rn(-0.1, rate, Y[u]);
      if (lane == 0) sv[li] = __fma_rn(0.7, rate, vi);
      const long long t4 = clk();
      __syncwarp();
      const long long t5 = clk();
      const double chk = sv[li];  // store -> load turnaround
      const long long t6 = clk() + (chk == 1e300 ? 1 : 0) + (Pl == 1e300 ? 1 : 0);
      acc[0] += t1 - t0;
      acc[1] += t2 - t1;
      acc[2] += t3 - t2;
      acc[3] += t4 - t3;
      acc[4] += t5 - t4;
      acc[5] += t6 - t5;
      acc[6] += t6 - t0;
    }
  }
  if (lane == 0)
    for (int k = 0; k < 7; ++k) out[k] = acc[k];
}

__global__ void lat(long long* out) {
  // dependent-chain latencies: LDS.64, SHFL (one 32-bit), DADD, DFMA
  __shared__ double s[64];
  __shared__ int si[64];
  const int lane = threadIdx.x;
  s[lane] = lane;
  s[lane + 32] = lane + 32;
  si[lane] = (lane + 1) & 31;
  si[lane + 32] = (lane + 1) & 31;
  __syncwarp();
  int idx = lane;
  long long t0 = clk();
  for (int i = 0; i < 256; ++i) idx = si[idx];
  long long t1 = clk();
  double x = s[idx];
  long long t2 = clk();
  for (int i = 0; i < 256; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1);
  long long t3 = clk();
  double y = x;
  for (int i = 0; i < 256; ++i) y = y + 1.0;
  long long t4 = clk();
  for (int i = 0; i < 256; ++i) y = __fma_rn(y, 1.0000001, 0.5);
  long long t5 = clk();
  int z = idx;
  for (int i = 0; i < 256; ++i) z = __shfl_xor_sync(0xffffffffu, z, 1);
  long long t6 = clk();
  if (lane == 0) {
    out[0] = (t1 - t0) / 256;
    out[1] = (t3 - t2) / 256;
    out[2] = (t4 - t3) / 256;
    out[3] = (t5 - t4) / 256;
    out[4] = (t6 - t5) / 256;
    out[5] = (long long)(y + z);
  }
}

int main() {
  static uint16_t h_nl[NP * CNT];
  static double h_pf[NP * CNT];
  srand(1);
  for (int k = 0; k < NP; ++k) {
    int used[S] = {0};
    used[200 + k] = 1;
    int s = 0;
    while (s < CNT) {
      int start = rand() % (S - 8), run = 2 + rand() % 5;
      for (int r = 0; r < run && s < CNT; ++r)
        if (!used[start + r]) {
          used[start + r] = 1;
          h_nl[k * CNT + s++] = (uint16_t)(start + r);
        }
    }
    for (int q = 0; q < CNT; ++q) h_pf[k * CNT + q] = -1e-3 * (1 + rand() % 100);
  }
  uint16_t* nl;
  double* pf;
  long long* out;
  cudaMalloc(&nl, sizeof(h_nl));
  cudaMalloc(&pf, sizeof(h_pf));
  cudaMalloc(&out, 16 * sizeof(long long));
  cudaMemcpy(nl, h_nl, sizeof(h_nl), cudaMemcpyHostToDevice);
  cudaMemcpy(pf, h_pf, sizeof(h_pf), cudaMemcpyHostToDevice);
  long long h[16];
  for (int w = 0; w < 2; ++w) lat<<<1, 32>>>(out);
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  printf("dependent latency (cycles): LDS.32 %lld  SHFL.f64(2x32) %lld  DADD %lld  DFMA %lld  SHFL.32 %lld\n", h[0],
         h[1], h[2], h[3], h[4]);
  for (int w = 0; w < 2; ++w) probe<<<1, 32>>>(nl, pf, out);
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[] = {"gathers + w", "partial + Y", "5-level shuffle", "rate + scatter issue", "syncwarp",
                         "store->load", "total"};
  for (int k = 0; k < 7; ++k) printf("%-22s %7.1f cycles/particle\n", names[k], double(h[k]) / (20 * NP));
  return 0;
}
