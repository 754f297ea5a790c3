// Device options of the C++ operator API (an addition to the reference's API; the reference
// runs on the CPU and has no counterpart).
//
// The operators of neighbors.hpp / damping.hpp / integrator.hpp run on the GPU over a device
// system kept resident per ReferenceNeighborhood (see csrc/host/resident.hpp): the CSR is uploaded
// once, every call moves only the particle fields the reference operator reads and writes.
#ifndef TLSPH_DEVICE_HPP
#define TLSPH_DEVICE_HPP

#include <vector>

#include "tlsph/particle_system.hpp"

namespace tlsph {

// Neighbour-sum order of the device kernels behind the operators:
//   Ordered (default): every sum is a left fold in the reference's slot order, so results equal
//            the reference arithmetic bit for bit (what the reference's own tests check);
//   Fast:    lane-parallel sums and the reassociated Gauss-Seidel update (within 1e-10 relative
//            L2 of Ordered; the throughput mode for production runs).
enum class Reduction { Ordered, Fast };

void set_operator_reduction(Reduction mode);
Reduction operator_reduction();

// Frees every resident device system (e.g. before building a much larger body).
void release_device_state();

// Page-locks the storage of a caller's ParticleSystem (and body-force array) so the operators'
// field transfers run as direct DMA (~55 GB/s per direction) instead of through a staging ring.
// The storage must not be reallocated or freed while pinned: call unpin_host_memory first.
template <int D>
void pin_host_memory(ParticleSystem<D>& system, std::vector<Vec<D>>* body = nullptr);
template <int D>
void unpin_host_memory(ParticleSystem<D>& system, std::vector<Vec<D>>* body = nullptr);

}  // namespace tlsph

#endif  // TLSPH_DEVICE_HPP
