// Staged 3^D cell stencils: the rows of a cell's stencil (x-runs of three
// cells, contiguous in cell-sorted order) and the padded tile layout shared by
// the damping sweep (sweep.cu) and the cell-tiled TL-SPH passes (tlsph.cu).
// Tile position of a stencil particle: rows are laid out one after another,
// each starting at the parity of its first global index (so 16-byte chunks
// of a row are aligned in both places); the per-slot index nloc (state.cu,
// k_nbr_fill / k_csr_from_ref) is that position.
#pragma once

#include "common.cuh"

namespace tlsph_cuda {

constexpr unsigned kFull = 0xffffffffu;


template <int D>
__host__ __device__ constexpr int seg_count() { return D == 2 ? 3 : 9; }

// Lane q < 3^(D-1) of the staging warp: particle extent [sstart, send) of stencil row q of cell c.
template <int D>
__device__ __forceinline__ void locate_row(const DFields& f, const int c[3], int lane, long long& sstart,
                                           long long& send) {
  sstart = 0;
  send = 0;
  if (lane < seg_count<D>()) {
    const int dy = (D == 2 ? lane : lane % 3) - 1;
    const int dz = D == 2 ? 0 : lane / 3 - 1;
    const int y = c[1] + dy;
    const int z = c[2] + dz;
    bool ok = y >= 0 && y < f.dims[1];
    if (D == 3) ok = ok && z >= 0 && z < f.dims[2];
    if (ok) {
      const int xlo = c[0] > 0 ? c[0] - 1 : 0;
      const int xhi = c[0] + 1 < f.dims[0] ? c[0] + 1 : f.dims[0] - 1;
      const long long row = D == 3 ? (static_cast<long long>(z) * f.dims[1] + y) * f.dims[0]
                                   : static_cast<long long>(y) * f.dims[0];
      sstart = f.cell_start[row + xlo];
      send = f.cell_start[row + xhi + 1];
    }
  }
}

// Stencil row table in registers: lane q < 3^(D-1) holds row q, as 16-byte
// pairs (the tile keeps every row at the parity of its global position).
struct RowPairs {
  long long gp;  // global index of the row's first pair (element 2 gp)
  int tp;        // tile index of the row's first pair
  int npair;     // pairs staged for the row
  int excl;      // exclusive prefix of npair over the rows
  int total;     // pairs over all rows
};

__device__ __forceinline__ RowPairs row_pairs(long long sstart, int slen, int sbase, int lane) {
  RowPairs r;
  const int par = static_cast<int>(sstart & 1);
  r.gp = (sstart - par) >> 1;
  r.tp = (sbase - par) >> 1;
  r.npair = slen > 0 ? (slen + par + 1) >> 1 : 0;
  int incl = r.npair;
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const int x = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += x;
  }
  r.excl = incl - r.npair;
  r.total = __shfl_sync(kFull, incl, 15);
  return r;
}

// For pair p of the flattened row table: its row q and offset in the row.
template <int D>
__device__ __forceinline__ void locate_pair(const RowPairs& r, int p, int& q, int& off) {
  q = 0;
#pragma unroll
  for (int k = 1; k < seg_count<D>(); ++k) q += p >= __shfl_sync(kFull, r.excl, k) ? 1 : 0;
  off = p - __shfl_sync(kFull, r.excl, q);
}

}  // namespace tlsph_cuda
