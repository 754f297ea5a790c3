// Per-kernel overhead of a chain of dependent launches (579 CTAs x 32 threads,
// as one cfg2 colour phase), plain stream order vs programmatic dependent launch,
// eager and captured in a CUDA graph.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pdl_bench tools/pdl_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* x, int pdl, int work) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  double a = x[blockIdx.x * 32 + threadIdx.x];
  for (int i = 0; i < work; ++i) a = a * 1.0000001 + 1e-9;
  x[blockIdx.x * 32 + threadIdx.x] = a;
}

void launch(cudaStream_t s, double* x, int pdl, int work) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(579);
  cfg.blockDim = dim3(32);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, x, pdl, work);
}

int main() {
  double* x;
  cudaMalloc(&x, 579 * 32 * sizeof(double));
  cudaMemset(x, 0, 579 * 32 * sizeof(double));
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int N = 540;
  for (int work : {0, 2000}) {
    for (int graph = 0; graph < 2; ++graph) {
      for (int pdl = 0; pdl < 2; ++pdl) {
        cudaGraphExec_t ge = nullptr;
        if (graph) {
          cudaGraph_t g;
          cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
          for (int i = 0; i < N; ++i) launch(s, x, pdl, work);
          cudaStreamEndCapture(s, &g);
          cudaGraphInstantiate(&ge, g, 0);
          cudaGraphDestroy(g);
        }
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
          cudaEventRecord(a, s);
          if (graph) cudaGraphLaunch(ge, s);
          else
            for (int i = 0; i < N; ++i) launch(s, x, pdl, work);
          cudaEventRecord(b, s);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (ms < best) best = ms;
        }
        printf("work %5d %-6s %-5s %7.2f us per kernel (%s)\n", work, graph ? "graph" : "eager", pdl ? "pdl" : "plain",
               best * 1e3 / N, cudaGetErrorString(cudaGetLastError()));
        if (ge) cudaGraphExecDestroy(ge);
      }
    }
  }
  return 0;
}
