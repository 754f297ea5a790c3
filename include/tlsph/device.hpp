// Device options of the C++ operator API (an addition to the reference's API; the reference
// runs on the CPU and has no counterpart).
//
// The operators of neighbors.hpp / damping.hpp / integrator.hpp run on the GPU over a device
// system kept resident per ReferenceNeighborhood (see csrc/host/resident.hpp): the CSR is uploaded
// once, every call moves only the particle fields the reference operator reads and writes.
#ifndef TLSPH_DEVICE_HPP
#define TLSPH_DEVICE_HPP

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

}  // namespace tlsph

#endif  // TLSPH_DEVICE_HPP
