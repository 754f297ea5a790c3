// FP64 issue throughput per SM sub-partition: one warp running 8 independent DFMA/DADD chains.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void tput(double* out, long long iters, long long* cycles) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.0 + 1e-9 * (threadIdx.x + k);
  const double y = 1.0000001, z = 1e-12;
  long long t0 = clock64();
  for (long long i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) a[k] = __fma_rn(a[k], y, z);
      if (OP == 1) a[k] = a[k] + y;
      if (OP == 2) a[k] = __shfl_xor_sync(0xffffffffu, a[k], 1);
      if (OP == 3) a[k] = __fmaf_rn(static_cast<float>(a[k]), 1.0f, 1e-7f);
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 8);
  const char* names[] = {"DFMA", "DADD", "SHFL(f64)", "FFMA(f32, cvt)"};
  for (int warps : {1, 4, 16}) {
    for (int op = 0; op < 3; ++op) {
      const long long iters = 4096;
      for (int r = 0; r < 2; ++r) {
        if (op == 0) tput<0><<<1, 32 * warps>>>(out, iters, cyc);
        if (op == 1) tput<1><<<1, 32 * warps>>>(out, iters, cyc);
        if (op == 2) tput<2><<<1, 32 * warps>>>(out, iters, cyc);
      }
      long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("warps/SM %2d %-10s %6.2f cycles per warp-instruction (per warp), %6.2f per SM\n", warps, names[op],
             double(c) / (iters * 8), double(c) / (iters * 8 * warps));
    }
  }
  return 0;
}
