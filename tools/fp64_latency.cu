// Microbenchmark: dependent-chain latencies on the B200 (one warp) for the
// instructions on the damping sweep's critical path (DADD, DMUL, DFMA,
// SHFL.BFLY of a double, LDS.64, MUFU-based double division).
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, const double* in, long long iters, long long* cycles) {
  __shared__ double sh[64];
  double x = in[threadIdx.x], y = in[threadIdx.x + 32];
  sh[threadIdx.x] = x;
  sh[threadIdx.x + 32] = y;
  __syncwarp();
  int idx = threadIdx.x;
  long long t0 = clock64();
  for (long long k = 0; k < iters; ++k) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (OP == 0) x = x + y;
      if (OP == 1) x = x * y;
      if (OP == 2) x = __fma_rn(x, y, y);
      if (OP == 3) x = __shfl_xor_sync(0xffffffffu, x, 1);
      if (OP == 4) { x = sh[idx]; idx = static_cast<int>(x) & 31; }
      if (OP == 5) x = y / x;
      if (OP == 6) { x = __shfl_xor_sync(0xffffffffu, x, 1) + x; }
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cycles = t1 - t0;
}

int main() {
  double *in, *out;
  long long* cyc;
  cudaMalloc(&in, 64 * sizeof(double));
  cudaMalloc(&out, 64 * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  double h[64];
  for (int i = 0; i < 64; ++i) h[i] = 1.0 + 1e-9 * i;
  h[0] = 0.0;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  const char* names[] = {"DADD", "DMUL", "DFMA", "SHFL(f64)", "LDS.64 (pointer chase)", "DDIV (IEEE)", "SHFL+DADD (reduce level)"};
  const long long iters = 4096;
  for (int op = 0; op < 7; ++op) {
    long long c = 0;
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: chain<0><<<1, 32>>>(out, in, iters, cyc); break;
        case 1: chain<1><<<1, 32>>>(out, in, iters, cyc); break;
        case 2: chain<2><<<1, 32>>>(out, in, iters, cyc); break;
        case 3: chain<3><<<1, 32>>>(out, in, iters, cyc); break;
        case 4: chain<4><<<1, 32>>>(out, in, iters, cyc); break;
        case 5: chain<5><<<1, 32>>>(out, in, iters, cyc); break;
        case 6: chain<6><<<1, 32>>>(out, in, iters, cyc); break;
      }
      cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    }
    printf("%-28s %7.2f cycles per dependent op\n", names[op], double(c) / (iters * 16));
  }
  return 0;
}
