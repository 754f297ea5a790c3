// Host<->device copy rates on this box: pageable vs pinned vs registered host memory, and the cost
// of cudaHostRegister itself (the operator API's per-call transfers read and write the caller's
// std::vector storage). nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/h2d_probe.cu -o tools/h2d_probe
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  const size_t sizes[] = {size_t(6) << 20, size_t(64) << 20, size_t(1) << 30};
  for (size_t bytes : sizes) {
    void* d = nullptr;
    cudaMalloc(&d, bytes);
    std::vector<char> pageable(bytes, 1);
    void* pinned = nullptr;
    cudaMallocHost(&pinned, bytes);
    std::memset(pinned, 1, bytes);
    auto rate = [&](void* h, bool h2d) {
      const int reps = bytes < (size_t(100) << 20) ? 20 : 4;
      cudaMemcpy(h2d ? d : h, h2d ? h : d, bytes, h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost);
      const double t0 = now();
      for (int k = 0; k < reps; ++k)
        cudaMemcpy(h2d ? d : h, h2d ? h : d, bytes, h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost);
      return bytes * reps / (now() - t0) / 1e9;
    };
    const double pg_h2d = rate(pageable.data(), true), pg_d2h = rate(pageable.data(), false);
    const double pn_h2d = rate(pinned, true), pn_d2h = rate(pinned, false);
    double t0 = now();
    cudaHostRegister(pageable.data(), bytes, cudaHostRegisterDefault);
    const double reg = now() - t0;
    const double rg_h2d = rate(pageable.data(), true), rg_d2h = rate(pageable.data(), false);
    t0 = now();
    cudaHostUnregister(pageable.data());
    const double unreg = now() - t0;
    // host memcpy into pinned (one thread)
    t0 = now();
    std::memcpy(pinned, pageable.data(), bytes);
    const double mc = bytes / (now() - t0) / 1e9;
    std::printf("{\"bytes\": %zu, \"pageable_h2d_gbs\": %.1f, \"pageable_d2h_gbs\": %.1f, \"pinned_h2d_gbs\": %.1f, "
                "\"pinned_d2h_gbs\": %.1f, \"registered_h2d_gbs\": %.1f, \"registered_d2h_gbs\": %.1f, "
                "\"register_ms\": %.3f, \"unregister_ms\": %.3f, \"memcpy_1thread_gbs\": %.1f}\n",
                bytes, pg_h2d, pg_d2h, pn_h2d, pn_d2h, rg_h2d, rg_d2h, reg * 1e3, unreg * 1e3, mc);
    cudaFreeHost(pinned);
    cudaFree(d);
  }
  return 0;
}
