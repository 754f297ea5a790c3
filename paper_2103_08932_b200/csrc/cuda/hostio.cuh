// Host <-> device copies of the caller's field arrays.
//
// The operator API moves ParticleSystem<D> fields that live in the caller's pageable std::vector
// storage every call. The driver's own pageable copies run at 11-18 GB/s on the GPU hosts, pinned
// DMA at ~55 GB/s (tools/h2d_probe, profiles/). Large pageable transfers therefore go through a
// small pinned ring: a team of host threads copies piece k+1 into the ring while the DMA engine
// moves piece k. Pinned sources/destinations and small transfers go straight to cudaMemcpyAsync.
// copy_to_device returns when the data is on the device side of the stream (later work on `st`
// sees it); copy_to_host returns when the data is in `dst`.
#ifndef TLSPH_CUDA_HOSTIO_CUH
#define TLSPH_CUDA_HOSTIO_CUH

#include <cuda_runtime.h>

#include <cstddef>

namespace tlsph_cuda {

void copy_to_device(void* dst, const void* src, size_t bytes, cudaStream_t st);
void copy_to_host(void* dst, const void* src, size_t bytes, cudaStream_t st);

}  // namespace tlsph_cuda

#endif  // TLSPH_CUDA_HOSTIO_CUH
