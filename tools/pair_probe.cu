// Cycles per pair step of the pairwise-split chain (one warp, lanes 0..2 one component each),
// with the sweep's shared-memory layout: variants isolate loads, stores and the fp64 chain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/pair_probe tools/pair_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int S = 512, CNT = 76, NP = 18;

template <int MODE>  // 0 full, 1 no stores, 2 chain only (operands from registers)
__global__ void pairs(const uint16_t* nl_g, double* out, long long* cyc, int reps) {
  __shared__ double sv[3][S];
  __shared__ double2 rec[NP * CNT];
  __shared__ uint16_t nl[NP * CNT];
  const int lane = threadIdx.x;
  for (int e = lane; e < S; e += 32)
    for (int d = 0; d < 3; ++d) sv[d][e] = 0.001 * e + d;
  for (int e = lane; e < NP * CNT; e += 32) {
    nl[e] = nl_g[e];
    rec[e] = make_double2(1e-3 * (1 + e % 7), (e % 13 == 0) ? -1.0 : 1.0);
  }
  __syncwarp();
  long long t0 = clock64();
  if (lane < 3) {
    double* vd = sv[lane];
    for (int rep = 0; rep < reps; ++rep) {
      for (int pk = 0; pk < NP; ++pk) {
        const int lo = pk * CNT, cnt = CNT;
        const int li = 200 + pk;
        const double mi = 1.0;
        double vi = vd[li];
        for (int pass = 0; pass < 2; ++pass) {
          for (int u0 = 0; u0 < cnt; u0 += 8) {
            int jb[8];
            double kb[8], mb[8], vjb[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int u = u0 + q < cnt ? u0 + q : cnt - 1;
              const int s = pass == 0 ? u : cnt - 1 - u;
              if (MODE == 2) {
                jb[q] = s;
                kb[q] = 1e-3 * q;
                mb[q] = 1.0;
                vjb[q] = 0.5 * q;
              } else {
                const int j = nl[lo + s];
                const double2 r = rec[lo + s];
                jb[q] = j;
                kb[q] = r.x;
                mb[q] = r.y;
                vjb[q] = vd[j];
              }
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              if (u0 + q >= cnt) break;
              const double scaled = kb[q] * (vi - vjb[q]);
              vi = vi + fabs(mb[q]) * scaled;
              if (MODE == 0 && mb[q] > 0.0) vd[jb[q]] = vjb[q] - mi * scaled;
            }
          }
        }
        vd[li] = vi;
      }
    }
  }
  long long t1 = clock64();
  if (lane == 0) {
    cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x] = sv[0][0] + sv[1][1];
  }
}

template <int MODE>
void run(const char* name, const uint16_t* nl, double* out, long long* cyc) {
  const int reps = 10;
  for (int blocks : {1, 148 * 4}) {
    for (int w = 0; w < 2; ++w) pairs<MODE><<<blocks, 32>>>(nl, out, cyc, reps);
    cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    printf("%-22s blocks %4d %7.1f cycles/pair step (%s)\n", name, blocks, double(c) / (reps * NP * 2 * CNT),
           cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  static uint16_t h[NP * CNT];
  srand(2);
  for (int k = 0; k < NP; ++k) {
    int used[S] = {0};
    used[200 + k] = 1;
    for (int s = 0; s < CNT; ++s) {
      int j;
      do j = rand() % S; while (used[j]);
      used[j] = 1;
      h[k * CNT + s] = (uint16_t)j;
    }
  }
  uint16_t* nl;
  double* out;
  long long* cyc;
  cudaMalloc(&nl, sizeof(h));
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMalloc(&cyc, 1024 * sizeof(long long));
  cudaMemcpy(nl, h, sizeof(h), cudaMemcpyHostToDevice);
  run<0>("full", nl, out, cyc);
  run<1>("no stores", nl, out, cyc);
  run<2>("chain only", nl, out, cyc);
  return 0;
}
