// Splitting cell-linked list through the device (reference:
// proj/src/tlsph/neighbors.cpp:14-174). build_cell_grid and
// build_reference_neighborhoods run the GPU counting sort / CSR fill
// (state.cu) and return the reference's host structures bit for bit;
// block_decompose and block_sweep are integer bookkeeping on the host.
#include "tlsph/neighbors.hpp"

#include <algorithm>
#include <cmath>
#include <string>

#include "devbridge.hpp"
#include "resident.hpp"
#include "tlsph/errors.hpp"

namespace tlsph {

template <int D>
std::array<int, D> CellGrid<D>::coords_of_position(const Vec<D>& p) const {
  std::array<int, D> c{};
  for (int d = 0; d < D; ++d) {
    const int idx = static_cast<int>(std::floor((p[d] - origin[d]) / cell_size));
    c[d] = std::clamp(idx, 0, dims[d] - 1);
  }
  return c;
}

template <int D>
CellGrid<D> build_cell_grid(std::span<const Vec<D>> positions, double cutoff) {
  require(!positions.empty(), ErrorKind::InvalidArgument, "cell grid needs at least one particle");
  require(cutoff > 0.0, ErrorKind::InvalidArgument, "cell grid cutoff must be positive");
  std::vector<double> flat(positions.size() * D);
  for (size_t i = 0; i < positions.size(); ++i)
    for (int d = 0; d < D; ++d) flat[i * D + d] = positions[i][d];
  host::DevHandle h;
  host::check(tlsph_dev_create_grid(D, positions.size(), flat.data(), cutoff, h.out()));
  int dims[3] = {1, 1, 1};
  double origin[3] = {0, 0, 0};
  double cell = 0.0;
  int64_t ncells = 0;
  host::check(tlsph_dev_grid_info(h.get(), dims, origin, &cell, &ncells));
  CellGrid<D> g;
  g.cell_size = cell;
  for (int d = 0; d < D; ++d) {
    g.dims[d] = dims[d];
    g.origin[d] = origin[d];
  }
  std::vector<int32_t> cell_of(positions.size()), parts(positions.size());
  std::vector<int64_t> start(static_cast<size_t>(ncells) + 1);
  host::check(tlsph_dev_grid_cells(h.get(), cell_of.data(), start.data(), parts.data()));
  g.cell_of.assign(cell_of.begin(), cell_of.end());
  g.cells.assign(static_cast<size_t>(ncells), {});
  for (int64_t c = 0; c < ncells; ++c) g.cells[c].assign(parts.begin() + start[c], parts.begin() + start[c + 1]);
  return g;
}

template <int D>
BlockDecomposition<D> block_decompose(const CellGrid<D>& grid) {
  BlockDecomposition<D> out;
  out.blocks.assign(ipow3(D), {});
  for (int cell = 0; cell < grid.cell_count(); ++cell) {
    const auto c = grid.coords_of(cell);
    int b = 0, stride = 1;
    for (int d = 0; d < D; ++d) {
      b += (c[d] % 3) * stride;
      stride *= 3;
    }
    out.blocks[static_cast<size_t>(b)].push_back(cell);
  }
  return out;
}

template <int D>
ReferenceNeighborhood<D> build_reference_neighborhoods(std::span<const Vec<D>> r0, std::span<const double> V0,
                                                       const SmoothingKernel& kernel, const CellGrid<D>& grid) {
  const size_t n = r0.size();
  require(V0.size() == n, ErrorKind::InvalidArgument, "volume array size does not match particle count");
  (void)grid;  // rebuilt on the device from the same r0 and cutoff
  std::vector<double> flat(n * D);
  for (size_t i = 0; i < n; ++i)
    for (int d = 0; d < D; ++d) flat[i * D + d] = r0[i][d];
  const std::vector<double> rho0(n, 1.0);
  host::DevHandle h;
  host::check(tlsph_dev_create(D, n, flat.data(), V0.data(), rho0.data(), nullptr, kernel.h(), h.out()));
  const int64_t S = tlsph_dev_slot_count(h.get());
  ReferenceNeighborhood<D> nbh;
  nbh.offsets.resize(n + 1);
  nbh.neighbor.resize(static_cast<size_t>(S));
  nbh.r0_len.resize(static_cast<size_t>(S));
  nbh.dwdr0.resize(static_cast<size_t>(S));
  nbh.pair_factor.resize(static_cast<size_t>(S));
  nbh.e0.resize(static_cast<size_t>(S));
  static_assert(sizeof(Vec<D>) == D * sizeof(double));
  host::check(tlsph_dev_get_neighborhood(h.get(), nbh.offsets.data(), nbh.neighbor.data(), nbh.r0_len.data(),
                                         reinterpret_cast<double*>(nbh.e0.data()), nbh.dwdr0.data(),
                                         nbh.pair_factor.data()));
  // the device system that built the CSR stays resident for the operators that will use it
  // (returned by value, the vectors keep their storage, so the registered identity holds)
  host::adopt<D>(std::move(h), nbh);
  return nbh;
}

template <int D>
void block_sweep(const BlockDecomposition<D>& blocks, const std::function<void(int, SweepDirection)>& cell_task,
                 SweepSchedule schedule, int threads) {
  (void)threads;  // same-colour tasks are independent; run in order here
  auto pass = [&](SweepDirection dir) {
    const int nb = static_cast<int>(blocks.blocks.size());
    for (int b = 0; b < nb; ++b) {
      const auto& cells = blocks.blocks[static_cast<size_t>(dir == SweepDirection::Forward ? b : nb - 1 - b)];
      const size_t nc = cells.size();
      for (size_t k = 0; k < nc; ++k) cell_task(cells[dir == SweepDirection::Forward ? k : nc - 1 - k], dir);
    }
  };
  pass(SweepDirection::Forward);
  if (schedule == SweepSchedule::ForwardThenReverse) pass(SweepDirection::Reverse);
}

template struct CellGrid<2>;
template struct CellGrid<3>;
template CellGrid<2> build_cell_grid<2>(std::span<const Vec<2>>, double);
template CellGrid<3> build_cell_grid<3>(std::span<const Vec<3>>, double);
template BlockDecomposition<2> block_decompose<2>(const CellGrid<2>&);
template BlockDecomposition<3> block_decompose<3>(const CellGrid<3>&);
template ReferenceNeighborhood<2> build_reference_neighborhoods<2>(std::span<const Vec<2>>, std::span<const double>,
                                                                   const SmoothingKernel&, const CellGrid<2>&);
template ReferenceNeighborhood<3> build_reference_neighborhoods<3>(std::span<const Vec<3>>, std::span<const double>,
                                                                   const SmoothingKernel&, const CellGrid<3>&);
template void block_sweep<2>(const BlockDecomposition<2>&, const std::function<void(int, SweepDirection)>&,
                             SweepSchedule, int);
template void block_sweep<3>(const BlockDecomposition<3>&, const std::function<void(int, SweepDirection)>&,
                             SweepSchedule, int);

}  // namespace tlsph
