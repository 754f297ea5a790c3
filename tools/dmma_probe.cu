// Microbenchmark: dependent latency of the chain's 3-component warp sum, the transposing shuffle
// butterfly (sweep_chain.cuh warp_sum_vec) against a sum through two fp64 MMAs (mma.sync m8n8k4).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2103_08932_b200/csrc/cuda/sweep_chain.cuh"

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(0.0), "d"(0.0));
}

// Sum over the 32 lanes of x[c], c < 3, result in every lane.
// MMA 1 (B = ones): D[r][*] = sum of lanes 4r..4r+3 (lane l gets its group's sum R[l/4]).
// Shuffle: lane 4 r2 + k fetches R[k + 4 (r2 & 1)] from lane 4 (k + 4 (r2 & 1)).
// MMA 2 (B = ones): D[r2][*] = sum_k R[k + 4 (r2 & 1)] = H[r2 & 1]; xor-4 add gives the total.
__device__ __forceinline__ void warp_sum3_mma(double (&x)[3], int lane) {
  const int src = 4 * ((lane & 3) + 4 * ((lane >> 2) & 1));
  double r[3], d1;
#pragma unroll
  for (int c = 0; c < 3; ++c) dmma(r[c], d1, x[c], 1.0);
#pragma unroll
  for (int c = 0; c < 3; ++c) r[c] = __shfl_sync(0xffffffffu, r[c], src);
#pragma unroll
  for (int c = 0; c < 3; ++c) dmma(r[c], d1, r[c], 1.0);
#pragma unroll
  for (int c = 0; c < 3; ++c) x[c] = r[c] + __shfl_xor_sync(0xffffffffu, r[c], 4);
}

// One MMA (groups of four lanes), then a three-level xor butterfly over the eight group sums.
__device__ __forceinline__ void warp_sum3_mma1(double (&x)[3], int lane) {
  double r[3], d1;
#pragma unroll
  for (int c = 0; c < 3; ++c) dmma(r[c], d1, x[c], 1.0);
#pragma unroll
  for (int o = 4; o < 32; o <<= 1)
#pragma unroll
    for (int c = 0; c < 3; ++c) r[c] += __shfl_xor_sync(0xffffffffu, r[c], o);
#pragma unroll
  for (int c = 0; c < 3; ++c) x[c] = r[c];
}

template <int MODE>
__global__ void probe(double* out, long long iters, long long* cyc) {
  const int lane = threadIdx.x;
  double x[3] = {1e-3 * lane, 2e-3 * lane + 1, 3e-3 * lane - 1};
  long long t0 = clock64();
  for (long long k = 0; k < iters; ++k) {
    if (MODE == 0) tlsph_cuda::warp_sum_vec<3>(x, lane);
    else if (MODE == 1) warp_sum3_mma(x, lane);
    else warp_sum3_mma1(x, lane);
#pragma unroll
    for (int c = 0; c < 3; ++c) x[c] = x[c] * (1.0 / 32.0) + 1e-3 * lane;  // keep it a chain
  }
  long long t1 = clock64();
  out[lane] = x[0] + x[1] + x[2];
  if (lane == 0) *cyc = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 64 * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  // correctness: one reduction of known values
  const long long it = 100000;
  for (int mode = 0; mode < 3; ++mode) {
    for (int w = 0; w < 2; ++w) {
      if (mode == 0) probe<0><<<1, 32>>>(out, it, cyc);
      else if (mode == 1) probe<1><<<1, 32>>>(out, it, cyc);
      else probe<2><<<1, 32>>>(out, it, cyc);
    }
    cudaDeviceSynchronize();
    long long c = 0;
    double o[32];
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
    printf("%s: %.1f cycles per reduction step (out[0]=%.17g out[31]=%.17g) %s\n", mode == 0 ? "shuffle tree" : mode == 1 ? "2x DMMA" : "DMMA + 3 xor levels",
           double(c) / it, o[0], o[31], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
