// Microbenchmark of k_sweep_fast's per-particle chain (one warp = one cell,
// all D components per lane, K slots per lane), on a synthetic stencil tile
// with the sweep's data layout. Variants isolate the cost of the metadata
// loads, the shuffle reduction and the scatter.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/chain_fast tools/chain_fast.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2103_08932_b200/csrc/cuda/sweep_chain.cuh"

constexpr int S = 512, NP = 18, K = 3, D = 3, CNT = 76;

struct Smem {
  double sv[D][S];
  double pf[NP * CNT];
  double qf[NP * CNT];
  uint16_t nl[NP * CNT];
  long long offs[NP + 2];
  double diag[NP], y[NP];
};

// MODE bits: 1 = skip shuffles, 2 = skip scatter stores
template <int MODE>
__global__ void __launch_bounds__(128) chain(const uint16_t* nloc, const double* pf, double* out, long long* cyc,
                                            int reps) {
  extern __shared__ __align__(16) unsigned char raw[];
  Smem& t = *reinterpret_cast<Smem*>(raw);
  const int lane = threadIdx.x;
  const int nthr = blockDim.x;
  for (int e = lane; e < S; e += nthr) {
    for (int d = 0; d < D; ++d) t.sv[d][e] = 0.001 * e + d;
  }
  for (int e = lane; e < NP * CNT; e += nthr) {
    t.nl[e] = nloc[e];
    t.pf[e] = pf[e];
    t.qf[e] = (nloc[e] % 97 == 5) ? 0.0 : pf[e] / (1.0 + nloc[e] * 1e-3);
  }
  if (lane <= NP) t.offs[lane] = lane * CNT;
  if (lane < NP) {
    t.diag[lane] = -1.0 - 0.01 * lane;
    t.y[lane] = 0.3;
  }
  __syncthreads();
  tlsph_cuda::ChainTile<D> ct;
  for (int d = 0; d < D; ++d) ct.sv[d] = t.sv[d];
  ct.pf = t.pf;
  ct.qf = t.qf;
  ct.nl = t.nl;
  ct.offs = t.offs;
  ct.s0 = 0;
  ct.diag = t.diag;
  ct.y = t.y;
  ct.lbase = 200;
  ct.np = NP;
  ct.forward = 1;
  ct.kb = 0.37;
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) tlsph_cuda::fast_chain<D, K, !(MODE & 1), !(MODE & 2)>(ct, lane);
  long long t1 = clock64();
  if (lane == 0) {
    cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x] = t.sv[0][0] + t.sv[1][1];
  }
}

template <int MODE>
void run(const char* name, const uint16_t* nl, const double* pf, double* out, long long* cyc) {
  const int reps = 40;
  const size_t smem = sizeof(Smem);
  cudaFuncSetAttribute(chain<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int blocks : {1, 148 * 4}) {
    const int threads = 32;
    for (int w = 0; w < 2; ++w) chain<MODE><<<blocks, threads, smem>>>(nl, pf, out, cyc, reps);
    cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    printf("%-28s blocks %4d %8.1f cycles/particle  (%s)\n", name, blocks, double(c) / (reps * NP),
           cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  static uint16_t h_nl[NP * CNT];
  static double h_pf[NP * CNT];
  srand(1);
  for (int k = 0; k < NP; ++k) {
    // neighbours: runs of consecutive stencil indices (as cell-sorted rows give), none equal to i
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
  double *pf, *out;
  long long* cyc;
  cudaMalloc(&nl, sizeof(h_nl));
  cudaMalloc(&pf, sizeof(h_pf));
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMalloc(&cyc, 1024 * sizeof(long long));
  cudaMemcpy(nl, h_nl, sizeof(h_nl), cudaMemcpyHostToDevice);
  cudaMemcpy(pf, h_pf, sizeof(h_pf), cudaMemcpyHostToDevice);
  run<0>("as k_sweep_fast", nl, pf, out, cyc);
  run<1>("no shuffles", nl, pf, out, cyc);
  run<2>("no scatter", nl, pf, out, cyc);
  run<3>("no shuffles, no scatter", nl, pf, out, cyc);
  return 0;
}
