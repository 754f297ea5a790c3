// TL-SPH elastic step on the fixed reference-configuration neighbour list.
//
// Reference: proj/src/tlsph/integrator.cpp:12-178, material.cpp:32-44.
//
// Neighbour sums use G lanes per particle: lane l folds slots l, l+G, ...
// in ascending order and the G partials are combined with xor shuffles.
// G = 1 (ORDERED mode) is exactly the reference's left fold over ascending
// reference j, so dF/dt, B0 and the momentum sum are bit-identical to the
// CPU arithmetic (the neo-Hookean log() differs from glibc by <= 1 ulp, so
// stresses, and everything downstream, are in the 1e-10 class).
//
// verlet_step is three fused passes (integrator.cpp:118-152):
//   A  per particle : density(J^n), half-kick F and r, constraints, P*B0
//   B  neighbour sum: momentum RHS, kick v, constraints
//   C  neighbour sum: dF/dt, density(J^{n+1/2}), half-kick F and r, constraints
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "system.cuh"
#include "tma.cuh"

namespace tlsph_cuda {

namespace {

unsigned grid_for(long long n, int block) { return static_cast<unsigned>((n + block - 1) / block); }

// ------------------------------------------------------------------ B0 (integrator.cpp:12-42)
template <int D>
__global__ void k_correction_matrices(DFields f, DScalars* sc) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= f.n || !is_owned(f, i)) return;  // a halo particle's neighbourhood is cut by the slab
  M<D> mom;
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int k = 0; k < D; ++k) mom.c[r][k] = 0.0;
  const long long lo = f.offs[i], hi = f.offs[i + 1];
  for (long long s = lo; s < hi; ++s) {
    const int j = f.nbr[s];
    const double w = -f.V0[j] * f.dwdr0[s] * f.r0_len[s];
    double e[D];
#pragma unroll
    for (int d = 0; d < D; ++d) e[d] = f.e0[d][s];
#pragma unroll
    for (int r = 0; r < D; ++r) {
      const double we = w * e[r];
#pragma unroll
      for (int k = 0; k < D; ++k) mom.c[r][k] = mom.c[r][k] + we * e[k];
    }
  }
  double sv[D];
  singular_values<D>(mom, sv);
  if (!(sv[D - 1] > 0.0) || sv[0] / sv[D - 1] > 1e8) {
    record_error(sc, ERR_DEGENERATE, static_cast<unsigned long long>(f.perm[i]));
    return;
  }
  store_mat<D>(f.B0, i, inverse(mom));
}

// ------------------------------------------------------------------ dF/dt (integrator.cpp:44-58)
// POST: fused tail of verlet pass C (density, half-kick, constraints).
// Neighbour passes B and C: each lane of a G-lane group handles TLSPH_TL_U (C) / TLSPH_TL_UB (B)
// slots per iteration with their loads issued together, and the kernels are held to 64
// registers (8 CTAs of 128 threads per SM). Measured on cfg3 (640,000 particles, 48.6 M slots):
// 1.206 -> 1.121 ms per elastic step; either change alone was neutral or slower (the batch
// needs registers, the bound alone costs spills). The macros remain for A/B builds.
#ifndef TLSPH_TL_U
#define TLSPH_TL_U 2
#endif
#ifndef TLSPH_TL_UB
#define TLSPH_TL_UB 2
#endif
#ifndef TLSPH_TL_LBB
#define TLSPH_TL_LBB 8
#endif
#ifndef TLSPH_TL_LBC
#define TLSPH_TL_LBC 8
#endif
#ifndef TLSPH_TL_GB3
#define TLSPH_TL_GB3 8
#endif
#ifndef TLSPH_TL_GC3
#define TLSPH_TL_GC3 8
#endif
constexpr int kGB3 = TLSPH_TL_GB3, kGC3 = TLSPH_TL_GC3;  // lanes per particle in 3D, passes B and C
#if TLSPH_TL_LBB > 0
#define TL_BOUNDS_B __launch_bounds__(128, TLSPH_TL_LBB)
#else
#define TL_BOUNDS_B
#endif
#if TLSPH_TL_LBC > 0
#define TL_BOUNDS_C __launch_bounds__(128, TLSPH_TL_LBC)
#else
#define TL_BOUNDS_C
#endif
// The ORDERED kernels (G = 1: one thread per particle, slot-order sums) are separate entry
// points with one slot per iteration and no register bound; both changes cost them ~20 %.

// Slot arrays of the neighbour passes: the FAST kernels (G > 1) read the rows in neighbour-index
// order (DFields::snbr, set up by k_sorted_rows), the ORDERED ones in the reference's order.
#ifndef TLSPH_TL_SORTED
#define TLSPH_TL_SORTED 1
#endif
template <int D, int G, bool OI = false>
// slots whose metadata and neighbour records a thread of the slot-order (OI) passes loads ahead of
// their (still strictly slot-ordered) accumulation
#ifndef TLSPH_TL_OU
#define TLSPH_TL_OU 1
#endif
#ifndef TLSPH_TL_STREAM_HINT
#define TLSPH_TL_STREAM_HINT 0
#endif
#ifndef TLSPH_TL_SLOTREC_HINT
#define TLSPH_TL_SLOTREC_HINT 0
#endif
struct SlotView {
  const int* nbr;
  const double* dw;
  const double* e0[D];
  __device__ explicit SlotView(const DFields& f) {
    const bool s = TLSPH_TL_SORTED && G > 1 && f.snbr;
    const bool o = OI;
    nbr = s ? f.snbr : o ? f.onbr : f.nbr;
    dw = s ? f.sdw : o ? f.odw : f.dwdr0;
#pragma unroll
    for (int d = 0; d < D; ++d) e0[d] = s ? f.se0[d] : o ? f.oe0[d] : f.e0[d];
  }
  // physical index of slot s of particle i (row start lo): the ORDERED (G == 1) passes read the
  // group-interleaved copy, slot k of particle i at ogbase[i / 32] + 32 k + i % 32
  __device__ __forceinline__ long long base(const DFields& f, long long i) const {
    return OI ? f.ogbase[i >> 5] + (i & 31) : 0;
  }
  __device__ __forceinline__ long long at(const DFields& f, long long ob, long long lo, long long s) const {
    if (OI) return ob + 32 * (s - lo);
    return s;
  }
  // Slot fields are read once per pass: streaming loads (evict-first in L1 and L2), so they do
  // not displace the neighbour records the gathers reuse (TLSPH_TL_STREAM_HINT=0: plain loads).
  __device__ __forceinline__ int nb(long long su) const { return TLSPH_TL_STREAM_HINT ? __ldcs(nbr + su) : nbr[su]; }
  __device__ __forceinline__ double w(long long su) const { return TLSPH_TL_STREAM_HINT ? __ldcs(dw + su) : dw[su]; }
  __device__ __forceinline__ double e(int d, long long su) const {
    return TLSPH_TL_STREAM_HINT ? __ldcs(e0[d] + su) : e0[d][su];
  }
  // (dW/dr0, e0) of slot su. 3D slot-order passes (TLSPH_TL_SLOTREC): one 32-byte record per slot
  // in the interleaved copy (build_ordered_rows), one 256-bit load instead of four 64-bit loads.
  __device__ __forceinline__ void load(long long su, double& dwv, double (&ev)[D]) const {
    if constexpr (OI && D == 3 && TLSPH_TL_SLOTREC) {
      // TLSPH_TL_SLOTREC_HINT (A/B): 1 = L1::no_allocate, 2 = + L2::evict_first, 3 = L1::evict_first
#if TLSPH_TL_SLOTREC_HINT == 1
      asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
#elif TLSPH_TL_SLOTREC_HINT == 2
      asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
#elif TLSPH_TL_SLOTREC_HINT == 3
      asm volatile("ld.global.nc.L1::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
#else
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
#endif
                   : "=d"(dwv), "=d"(ev[0]), "=d"(ev[1]), "=d"(ev[2])
                   : "l"(dw + 4 * su));
    } else {
      dwv = w(su);
#pragma unroll
      for (int d = 0; d < D; ++d) ev[d] = e(d, su);
    }
  }
};

// PDL (FAST passes B and C): launched with programmatic stream serialization, the kernel lets
// the next pass launch early and waits for the previous one before reading its output.
#ifndef TLSPH_TL_PDL
#define TLSPH_TL_PDL 1
#endif
// UV0: every reference volume equals f.v0_uniform, so the neighbour's V0 is not gathered
template <int D, int G, int U, bool POST, bool UV0 = false, bool OI = false>
__device__ __forceinline__ void deformation_rate_body(const DFields& f, DScalars* sc, double dt, int loop) {
  if (TLSPH_TL_PDL && G > 1) grid_dependency_wait();  // v of pass B's kick, F of pass A
  if (loop && sc->halt) return;
  const double half = 0.5 * (loop ? sc->dt : dt);
  const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long i = tid / G;
  const int l = static_cast<int>(tid % G);
  const bool active = i < f.n && is_owned(f, i);
  const SlotView<D, G, OI> sv(f);
  double rate[D][D];
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int q = 0; q < D; ++q) rate[r][q] = 0.0;
  if (active) {
    double vi[D];
#pragma unroll
    for (int d = 0; d < D; ++d) vi[d] = f.v[d][i];
    const long long hi = f.offs[i + 1], lo_i = f.offs[i], ob_i = sv.base(f, i);
    // U slots per lane per iteration: their loads and gathers are issued together (more bytes in
    // flight per thread); the lane still accumulates its slots in ascending order
    for (long long s = f.offs[i] + l; s < hi; s += U * G) {
      int j[U];
      double dw[U], e[U][D], vj[U][D], v0[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool ok = s + u * G < hi;
        const long long su = sv.at(f, ob_i, lo_i, ok ? s + u * G : s);
        j[u] = sv.nb(su);
        sv.load(su, dw[u], e[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if constexpr (OI && D == 3 && TLSPH_TL_V4) {
          // (v_j, V0_j) as one 32-byte record (k_pack_v4, launched before this pass): one 256-bit
          // gather instead of three or four 64-bit ones
          asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                       : "=d"(vj[u][0]), "=d"(vj[u][1]), "=d"(vj[u][2]), "=d"(v0[u])
                       : "l"(f.v4 + 4 * static_cast<long long>(j[u])));
        } else {
          v0[u] = UV0 ? f.v0_uniform : f.V0[j[u]];
#pragma unroll
          for (int d = 0; d < D; ++d) vj[u][d] = f.v[d][j[u]];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (u > 0 && s + u * G >= hi) break;
        const double k = v0[u] * dw[u];
#pragma unroll
        for (int r = 0; r < D; ++r) {
          const double kv = k * (vi[r] - vj[u][r]);
#pragma unroll
          for (int q = 0; q < D; ++q) rate[r][q] = rate[r][q] - kv * e[u][q];
        }
      }
    }
  }
  if (G > 1) {
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int q = 0; q < D; ++q) rate[r][q] = group_sum_fast<G>(rate[r][q]);
  }
  if (!active || l != 0) return;
  M<D> R;
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int q = 0; q < D; ++q) R.c[r][q] = rate[r][q];
  const M<D> dF = matmul(R, load_mat<D>(f.B0, i));
  store_mat<D>(f.dFdt, i, dF);
  if (POST) {
    M<D> F = load_mat<D>(f.F, i);
    const double J = det(F);
    if (!(J > 0.0)) record_error(sc, ERR_DENSITY_POST, static_cast<unsigned long long>(f.perm[i]));
    else f.rho[i] = f.rho0[i] / J;
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int q = 0; q < D; ++q) F.c[r][q] = F.c[r][q] + half * dF.c[r][q];
    store_mat<D>(f.F, i, F);
    if (f.flag[i]) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        f.v[d][i] = 0.0;
        f.r[d][i] = f.r0[d][i];
      }
    } else {
#pragma unroll
      for (int d = 0; d < D; ++d) f.r[d][i] = f.r[d][i] + half * f.v[d][i];
    }
  }
}

// (v, V0) of every particle as one 32-byte record for the 3D slot-order pass C's gathers; run
// right before that pass (v is final then: pass B's kick, and in a slab the halo refresh).
__global__ void k_pack_v4(DFields f) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= f.n) return;
  *reinterpret_cast<double4*>(f.v4 + 4 * i) = make_double4(f.v[0][i], f.v[1][i], f.v[2][i], f.V0[i]);
}

template <int D, int G, bool POST, bool UV0 = false>
__global__ void TL_BOUNDS_C k_deformation_rate(DFields f, DScalars* sc, double dt, int loop) {
  deformation_rate_body<D, G, TLSPH_TL_U, POST, UV0>(f, sc, dt, loop);
}
// register bound of the slot-order (one thread per particle) passes: minimum resident 128-thread
// blocks per SM (0: none; the compiler's choice, 70-72 registers = 7 blocks)
#ifndef TLSPH_TL_OMINB
#define TLSPH_TL_OMINB 0
#endif
#if TLSPH_TL_OMINB > 0
#define TL_BOUNDS_O __launch_bounds__(128, TLSPH_TL_OMINB)
#else
#define TL_BOUNDS_O
#endif
template <int D, bool POST, bool OI = false>
__global__ void TL_BOUNDS_O k_deformation_rate_ordered(DFields f, DScalars* sc, double dt, int loop) {
  deformation_rate_body<D, 1, OI ? TLSPH_TL_OU : 1, POST, false, OI>(f, sc, dt, loop);
}

// ------------------------------------------------------------------ density (integrator.cpp:60-78)
template <int D>
__global__ void k_update_density(DFields f, DScalars* sc) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= f.n || !is_owned(f, i)) return;
  const double J = det(load_mat<D>(f.F, i));
  if (!(J > 0.0)) {
    record_error(sc, ERR_DENSITY_PRE, static_cast<unsigned long long>(f.perm[i]));
    return;
  }
  f.rho[i] = f.rho0[i] / J;
}

// ------------------------------------------------------------------ stress term P*B0 (integrator.cpp:86-103)
// PRE: fused head of verlet pass A (density from J^n, half-kick, constraints).
template <int D, bool PRE>
__global__ void k_stress(DFields f, DScalars* sc, DMaterial mat, double dt, int loop) {
  if (TLSPH_TL_PDL) grid_launch_dependents();  // pass B may launch and wait
  if (loop && sc->halt) return;
  const double half = 0.5 * (loop ? sc->dt : dt);
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= f.n || !is_owned(f, i)) return;  // a slab's halo records arrive from their owner
  M<D> F = load_mat<D>(f.F, i);
  if (PRE) {
    const double J0 = det(F);
    if (!(J0 > 0.0)) record_error(sc, ERR_DENSITY_PRE, static_cast<unsigned long long>(f.perm[i]));
    else f.rho[i] = f.rho0[i] / J0;
    const M<D> dF = load_mat<D>(f.dFdt, i);
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int q = 0; q < D; ++q) F.c[r][q] = F.c[r][q] + half * dF.c[r][q];
    store_mat<D>(f.F, i, F);
    if (f.flag[i]) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        f.v[d][i] = 0.0;
        f.r[d][i] = f.r0[d][i];
      }
    } else {
#pragma unroll
      for (int d = 0; d < D; ++d) f.r[d][i] = f.r[d][i] + half * f.v[d][i];
    }
  }
  const double J = det(F);
  M<D> PB;
  if (!(J > 0.0)) {
    record_error(sc, ERR_MOMENTUM, static_cast<unsigned long long>(f.perm[i]));
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int q = 0; q < D; ++q) PB.c[r][q] = 0.0;
  } else {
    const M<D> S = second_pk<D>(F, J, mat);
    PB = matmul(matmul(F, S), load_mat<D>(f.B0, i));
  }
  // packed record for the momentum gather: P B0 row-major, then V0, 16-byte chunks (common.cuh)
  constexpr int W = pbv_stride<D>();
  double rec[W];
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int q = 0; q < D; ++q) rec[r * D + q] = PB.c[r][q];
  rec[D * D] = f.V0[i];
#pragma unroll
  for (int c = D * D + 1; c < W; ++c) rec[c] = 0.0;
#pragma unroll
  for (int k = 0; k < W / 2; ++k)
    *reinterpret_cast<double2*>(f.pbv + pbv_at<D>(f.n, i, 2 * k)) = make_double2(rec[2 * k], rec[2 * k + 1]);
}

// ------------------------------------------------------------------ momentum RHS (integrator.cpp:105-115)
// KICK: fused tail of verlet pass B (v += dt a, constraints).
// momentum_rhs's last steps for particle i from its neighbour sum acc (integrator.cpp:111-115):
// a = acc / m + ExternalAccel::eval (forces.hpp:34-38: body[i], + the contact plane at the current
// position); with KICK the loop's fused kick v += dt a and the constraints.
// PACK (3D, with KICK): also writes the particle's (v, V0) record for pass C's gathers (k_pack_v4's
// work, when pass C follows on the same stream with nothing touching v in between).
template <int D, bool KICK, bool PACK = false>
__device__ __forceinline__ void momentum_finish(const DFields& f, long long i, const double (&acc)[D], double dt,
                                                double v0i = 0.0) {
  const double mi = f.m[i];
  // ExternalAccel::eval (forces.hpp:34-38): body[i] (+ contact plane at the current position)
  double ext[D];
#pragma unroll
  for (int d = 0; d < D; ++d) ext[d] = f.body[d][i];
  if (f.contact) {
    double gap = (f.r[0][i] - f.cp_point[0]) * f.cp_normal[0];
#pragma unroll
    for (int d = 1; d < D; ++d) gap = gap + (f.r[d][i] - f.cp_point[d]) * f.cp_normal[d];
    const double kc = gap >= 0.0 ? 0.0 : f.cp_k * (-gap) / mi;
#pragma unroll
    for (int d = 0; d < D; ++d) ext[d] = ext[d] + (gap >= 0.0 ? 0.0 : kc * f.cp_normal[d]);
  }
  double a[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    a[d] = acc[d] / mi + ext[d];
    f.a[d][i] = a[d];
  }
  if (KICK) {
    double vn[D];
    if (f.flag[i]) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        vn[d] = 0.0;
        f.v[d][i] = 0.0;
        f.r[d][i] = f.r0[d][i];
      }
    } else {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        vn[d] = f.v[d][i] + dt * a[d];
        f.v[d][i] = vn[d];
      }
    }
    if constexpr (PACK && D == 3)
      *reinterpret_cast<double4*>(f.v4 + 4 * i) = make_double4(vn[0], vn[1], vn[2], v0i);
  }
}

template <int D, int G, int U, bool KICK, bool OI = false, bool PACK = false>
__device__ __forceinline__ void momentum_body(const DFields& f, DScalars* sc, double dt_arg, int loop) {
  if (TLSPH_TL_PDL && G > 1) {
    grid_launch_dependents();  // pass C may launch and wait
    grid_dependency_wait();    // pass A's records
  }
  if (loop && sc->halt) return;
  const double dt = loop ? sc->dt : dt_arg;
  const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long i = tid / G;
  const int l = static_cast<int>(tid % G);
  const bool active = i < f.n && is_owned(f, i);
  const SlotView<D, G, OI> sv(f);
  double acc[D];
#pragma unroll
  for (int d = 0; d < D; ++d) acc[d] = 0.0;
  if (active) {
    constexpr int W = pbv_stride<D>();
    double pbi[W];
    {
#pragma unroll
      for (int k = 0; k < W / 2; ++k) {
        const double2 x = *reinterpret_cast<const double2*>(f.pbv + pbv_at<D>(f.n, i, 2 * k));
        pbi[2 * k] = x.x;
        pbi[2 * k + 1] = x.y;
      }
    }
    const double V0i = pbi[D * D];
    const long long hi = f.offs[i + 1], lo_i = f.offs[i], ob_i = sv.base(f, i);
    for (long long s = f.offs[i] + l; s < hi; s += U * G) {
      int j[U];
      double dw[U], e[U][D];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long su = sv.at(f, ob_i, lo_i, s + u * G < hi ? s + u * G : s);
        j[u] = sv.nb(su);
        sv.load(su, dw[u], e[u]);
      }
      // P B0 and V0 of each j in W/2 16-byte loads from one packed record; all U records are
      // requested before the first is used (slots past the row end re-read a valid record)
      double pbj[U][W];
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int k = 0; k < W / 2; ++k) {
#ifdef TLSPH_PROBE_NOGATHER  // measurement probe only: the pass without its neighbour-record gather
          const double2 x = make_double2(pbi[2 * k] + j[u], pbi[2 * k + 1]);
#else
          if (D == 3 && TLSPH_PBV_WIDE) break;  // gathered below
          const double2 x = __ldg(reinterpret_cast<const double2*>(f.pbv + pbv_at<D>(f.n, j[u], 2 * k)));
#endif
          pbj[u][2 * k] = x.x;
          pbj[u][2 * k + 1] = x.y;
        }
#ifndef TLSPH_PROBE_NOGATHER
        if constexpr (D == 3 && TLSPH_PBV_WIDE) pbv_gather3(f.pbv, f.n, j[u], pbj[u]);
#endif
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (u > 0 && s + u * G >= hi) break;
        const double k = V0i * pbj[u][D * D] * dw[u];
#pragma unroll
        for (int r = 0; r < D; ++r) {
          double t = (k * (pbi[r * D] + pbj[u][r * D])) * e[u][0];
#pragma unroll
          for (int q = 1; q < D; ++q) t = t + (k * (pbi[r * D + q] + pbj[u][r * D + q])) * e[u][q];
          acc[r] = acc[r] + t;
        }
      }
    }
  }
  if (G > 1) {
#pragma unroll
    for (int d = 0; d < D; ++d) acc[d] = group_sum_fast<G>(acc[d]);
  }
  if (!active || l != 0) return;
  if constexpr (PACK) momentum_finish<D, KICK, true>(f, i, acc, dt, f.V0[i]);
  else momentum_finish<D, KICK>(f, i, acc, dt);
}

template <int D, int G, bool KICK>
__global__ void TL_BOUNDS_B k_momentum(DFields f, DScalars* sc, double dt_arg, int loop) {
  momentum_body<D, G, TLSPH_TL_UB, KICK>(f, sc, dt_arg, loop);
}
template <int D, bool KICK, bool OI = false, bool PACK = false>
__global__ void TL_BOUNDS_O k_momentum_ordered(DFields f, DScalars* sc, double dt_arg, int loop) {
  momentum_body<D, 1, OI ? TLSPH_TL_OU : 1, KICK, OI, PACK>(f, sc, dt_arg, loop);
}

template <int D>
__global__ void k_apply_constraints(DFields f) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= f.n || !f.flag[i]) return;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    f.v[d][i] = 0.0;
    f.r[d][i] = f.r0[d][i];
  }
}

// ------------------------------------------------------------------ reductions
// |v|max, |a|max (stable_dt, integrator.cpp:154-169), first non-finite
// particle (check_finite, runner.cpp:233-247) and kinetic energy partials
// (integrator.cpp:171-178).
template <int D>
__global__ void k_reduce(DFields f, double* __restrict__ partials, DScalars* sc, int want_ke) {
  __shared__ double s_v[256], s_a[256], s_k[256];
  double vmax = 0.0, amax = 0.0, ke = 0.0;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < f.n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (!is_owned(f, i)) continue;
    double sv = f.v[0][i] * f.v[0][i], sa = f.a[0][i] * f.a[0][i];
    bool fin = isfinite(f.v[0][i]) && isfinite(f.r[0][i]);
#pragma unroll
    for (int d = 1; d < D; ++d) {
      sv = sv + f.v[d][i] * f.v[d][i];
      sa = sa + f.a[d][i] * f.a[d][i];
      fin = fin && isfinite(f.v[d][i]) && isfinite(f.r[d][i]);
    }
    vmax = fmax(vmax, sqrt(sv));
    amax = fmax(amax, sqrt(sa));
    if (want_ke) ke += 0.5 * f.m[i] * sv;
    if (!fin) record_error(sc, ERR_NAN, static_cast<unsigned long long>(f.perm[i]));
  }
  s_v[threadIdx.x] = vmax;
  s_a[threadIdx.x] = amax;
  s_k[threadIdx.x] = ke;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (threadIdx.x < off) {
      s_v[threadIdx.x] = fmax(s_v[threadIdx.x], s_v[threadIdx.x + off]);
      s_a[threadIdx.x] = fmax(s_a[threadIdx.x], s_a[threadIdx.x + off]);
      s_k[threadIdx.x] += s_k[threadIdx.x + off];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partials[blockIdx.x * 3 + 0] = s_v[0];
    partials[blockIdx.x * 3 + 1] = s_a[0];
    partials[blockIdx.x * 3 + 2] = s_k[0];
  }
}

}  // namespace

// ====================================================================== host side
namespace {
template <typename Fn2, typename Fn3>
void dispatch(int D, Fn2&& f2, Fn3&& f3) {
  if (D == 2) f2();
  else f3();
}
}  // namespace

void DevSystem::correction_matrices() {
  reset_errors();
  DFields f = fields();
  dispatch(D, [&] { k_correction_matrices<2><<<grid_for(n, 128), 128, 0, stream>>>(f, scal.p); },
           [&] { k_correction_matrices<3><<<grid_for(n, 128), 128, 0, stream>>>(f, scal.p); });
  CK_LAUNCH("k_correction_matrices");
  raise_if_failed("compute_correction_matrices");
}

void DevSystem::deformation_rate() {
  DFields f = fields();
  // bodies with the group-interleaved slot copy run the slot-order kernels in both modes, as the
  // loop does (enqueue_verlet_pass): the standalone operator matches the loop bit for bit
  const bool ord = reduction == TLSPH_REDUCTION_ORDERED || f.onbr;
  if (D == 2) {
    if (ord) {
      if (f.onbr) k_deformation_rate_ordered<2, false, true><<<grid_for(n, 128), 128, 0, stream>>>(f, scal.p, 0.0, 0);
      else k_deformation_rate_ordered<2, false><<<grid_for(n, 128), 128, 0, stream>>>(f, scal.p, 0.0, 0);
    }
    else k_deformation_rate<2, 4, false><<<grid_for(n * 4, 128), 128, 0, stream>>>(f, scal.p, 0.0, 0);
  } else {
    if (ord) {
      if (f.onbr && TLSPH_TL_V4) k_pack_v4<<<grid_for(n, 256), 256, 0, stream>>>(f);
      if (f.onbr) k_deformation_rate_ordered<3, false, true><<<grid_for(n, 128), 128, 0, stream>>>(f, scal.p, 0.0, 0);
      else k_deformation_rate_ordered<3, false><<<grid_for(n, 128), 128, 0, stream>>>(f, scal.p, 0.0, 0);
    }
    else k_deformation_rate<3, kGC3, false><<<grid_for(n * kGC3, 128), 128, 0, stream>>>(f, scal.p, 0.0, 0);
  }
  CK_LAUNCH("k_deformation_rate");
  sync();
}

void DevSystem::update_density() {
  reset_errors();
  DFields f = fields();
  dispatch(D, [&] { k_update_density<2><<<grid_for(n, 256), 256, 0, stream>>>(f, scal.p); },
           [&] { k_update_density<3><<<grid_for(n, 256), 256, 0, stream>>>(f, scal.p); });
  CK_LAUNCH("k_update_density");
  raise_if_failed("update_density");
}

void DevSystem::momentum_rhs(const DMaterial& mat) {
  reset_errors();
  DFields f = fields();
  bool ord = reduction == TLSPH_REDUCTION_ORDERED;
  dispatch(D, [&] { k_stress<2, false><<<grid_for(n, 128), 128, 0, stream>>>(f, scal.p, mat, 0.0, 0); },
           [&] { k_stress<3, false><<<grid_for(n, 128), 128, 0, stream>>>(f, scal.p, mat, 0.0, 0); });
  CK_LAUNCH("k_stress");
  raise_if_failed("compute_momentum_rhs");  // the reference throws before the pair loop
  ord = ord || f.onbr;  // as deformation_rate: the loop's kernels wherever the interleaved copy exists
  if (D == 2) {
    if (ord) {
      if (f.onbr) k_momentum_ordered<2, false, true><<<grid_for(n, 128), 128, 0, stream>>>(f, scal.p, 0.0, 0);
      else k_momentum_ordered<2, false><<<grid_for(n, 128), 128, 0, stream>>>(f, scal.p, 0.0, 0);
    }
    else k_momentum<2, 4, false><<<grid_for(n * 4, 128), 128, 0, stream>>>(f, scal.p, 0.0, 0);
  } else {
    if (ord) {
      if (f.onbr) k_momentum_ordered<3, false, true><<<grid_for(n, 128), 128, 0, stream>>>(f, scal.p, 0.0, 0);
      else k_momentum_ordered<3, false><<<grid_for(n, 128), 128, 0, stream>>>(f, scal.p, 0.0, 0);
    }
    else k_momentum<3, kGB3, false><<<grid_for(n * kGB3, 128), 128, 0, stream>>>(f, scal.p, 0.0, 0);
  }
  CK_LAUNCH("k_momentum");
  sync();
}

// Enqueues one verlet pass (0: A, 1: B, 2: C) on the handle's stream (no sync).
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), long long threads, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid_for(threads, 128));
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = TLSPH_TL_PDL ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, kernel, args...));
}

// fused: the three passes are enqueued back to back on an undivided body (enqueue_verlet): pass B
// writes pass C's (v, V0) records itself (TLSPH_TL_PACK_IN_B) and k_pack_v4 is not launched; the
// per-pass entry of the x-slab driver refreshes halo velocities between B and C and packs after that.
#ifndef TLSPH_TL_PACK_IN_B
#define TLSPH_TL_PACK_IN_B 1
#endif
void enqueue_verlet_pass(DevSystem& s, const DMaterial& mat, double dt, int loop, int pass, bool fused = false) {
  DFields f = s.fields();
  const bool pack_in_b = fused && TLSPH_TL_PACK_IN_B && TLSPH_TL_V4 && f.onbr && !f.own && s.D == 3;
  const long long n = s.n;
  // large bodies (group-interleaved slot copy present): both modes run the slot-order one-thread
  // kernels (build_ordered_rows, state.cu); TLSPH_TL_EIGHT_LANES=1 keeps FAST on eight lanes (A/B)
  static const bool eight_lanes = [] {
    const char* e = std::getenv("TLSPH_TL_EIGHT_LANES");
    return e && *e == '1';
  }();
  const bool ord = s.reduction == TLSPH_REDUCTION_ORDERED || (f.onbr && !eight_lanes);
  cudaStream_t st = s.stream;
  if (s.D == 2) {
    if (pass == 0) k_stress<2, true><<<grid_for(n, 128), 128, 0, st>>>(f, s.scal.p, mat, dt, loop);
    else if (pass == 1 && ord) {
      if (f.onbr) k_momentum_ordered<2, true, true><<<grid_for(n, 128), 128, 0, st>>>(f, s.scal.p, dt, loop);
      else k_momentum_ordered<2, true><<<grid_for(n, 128), 128, 0, st>>>(f, s.scal.p, dt, loop);
    }
    else if (pass == 1) launch_pdl(k_momentum<2, 4, true>, n * 4, st, f, s.scal.p, dt, loop);
    else if (ord) {
      if (f.onbr) k_deformation_rate_ordered<2, true, true><<<grid_for(n, 128), 128, 0, st>>>(f, s.scal.p, dt, loop);
      else k_deformation_rate_ordered<2, true><<<grid_for(n, 128), 128, 0, st>>>(f, s.scal.p, dt, loop);
    }
    else if (f.v0_uniform > 0.0) launch_pdl(k_deformation_rate<2, 4, true, true>, n * 4, st, f, s.scal.p, dt, loop);
    else launch_pdl(k_deformation_rate<2, 4, true>, n * 4, st, f, s.scal.p, dt, loop);
  } else {
    if (pass == 0) k_stress<3, true><<<grid_for(n, 128), 128, 0, st>>>(f, s.scal.p, mat, dt, loop);
    else if (pass == 1 && ord) {
      if (pack_in_b) k_momentum_ordered<3, true, true, true><<<grid_for(n, 128), 128, 0, st>>>(f, s.scal.p, dt, loop);
      else if (f.onbr) k_momentum_ordered<3, true, true><<<grid_for(n, 128), 128, 0, st>>>(f, s.scal.p, dt, loop);
      else k_momentum_ordered<3, true><<<grid_for(n, 128), 128, 0, st>>>(f, s.scal.p, dt, loop);
    }
    else if (pass == 1) launch_pdl(k_momentum<3, kGB3, true>, n * kGB3, st, f, s.scal.p, dt, loop);
    else if (ord) {
      if (f.onbr && TLSPH_TL_V4 && !pack_in_b) k_pack_v4<<<grid_for(n, 256), 256, 0, st>>>(f);
      if (f.onbr) k_deformation_rate_ordered<3, true, true><<<grid_for(n, 128), 128, 0, st>>>(f, s.scal.p, dt, loop);
      else k_deformation_rate_ordered<3, true><<<grid_for(n, 128), 128, 0, st>>>(f, s.scal.p, dt, loop);
    }
    else if (f.v0_uniform > 0.0)
      launch_pdl(k_deformation_rate<3, kGC3, true, true>, n * kGC3, st, f, s.scal.p, dt, loop);
    else launch_pdl(k_deformation_rate<3, kGC3, true>, n * kGC3, st, f, s.scal.p, dt, loop);
  }
}

// Enqueues the three verlet passes on the handle's stream (no sync).
void enqueue_verlet(DevSystem& s, const DMaterial& mat, double dt, int loop) {
  for (int pass = 0; pass < 3; ++pass) enqueue_verlet_pass(s, mat, dt, loop, pass, true);
  CK_LAUNCH("verlet passes");
}

void DevSystem::verlet_step(const DMaterial& mat, double dt) {
  reset_errors();
  enqueue_verlet(*this, mat, dt, 0);
  raise_if_failed("verlet_step");
}

// One pass of verlet_step (x-slab driver: halo exchanges between the passes).
void DevSystem::verlet_pass(const DMaterial& mat, double dt, int pass) {
  if (pass < 0 || pass > 2) throw DevError(TLSPH_ERR_INVALID_ARGUMENT, "verlet pass must be 0 (A), 1 (B) or 2 (C)");
  reset_errors();
  enqueue_verlet_pass(*this, mat, dt, 0, pass);
  CK_LAUNCH("verlet pass");
  raise_if_failed("verlet_step");
}


void DevSystem::apply_constraints() {
  DFields f = fields();
  dispatch(D, [&] { k_apply_constraints<2><<<grid_for(n, 256), 256, 0, stream>>>(f); },
           [&] { k_apply_constraints<3><<<grid_for(n, 256), 256, 0, stream>>>(f); });
  CK_LAUNCH("k_apply_constraints");
  sync();
}

namespace {
struct Reduced {
  double vmax, amax, ke;
};

Reduced reduce_state(DevSystem& s, bool want_ke) {
  const unsigned nb = std::min<unsigned>(592, grid_for(s.n, 256));
  s.red.alloc(nb * 3);
  DFields f = s.fields();
  if (s.D == 2) k_reduce<2><<<nb, 256, 0, s.stream>>>(f, s.red.p, s.scal.p, want_ke ? 1 : 0);
  else k_reduce<3><<<nb, 256, 0, s.stream>>>(f, s.red.p, s.scal.p, want_ke ? 1 : 0);
  CK_LAUNCH("k_reduce");
  std::vector<double> hp(nb * 3);
  CK(cudaMemcpyAsync(hp.data(), s.red.p, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, s.stream));
  s.sync();
  Reduced r{0.0, 0.0, 0.0};
  for (unsigned b = 0; b < nb; ++b) {
    r.vmax = std::max(r.vmax, hp[b * 3]);
    r.amax = std::max(r.amax, hp[b * 3 + 1]);
    r.ke += hp[b * 3 + 2];
  }
  return r;
}
}  // namespace

double DevSystem::stable_dt(const DMaterial& mat, double h_) {
  reset_errors();
  const Reduced r = reduce_state(*this, false);
  reset_errors();  // stable_dt itself never fails
  double bound = h_ / (mat.c + r.vmax);
  if (r.amax > 0.0) bound = std::min(bound, std::sqrt(h_ / r.amax));
  return 0.6 * bound;
}

double DevSystem::kinetic_energy() {
  reset_errors();
  const Reduced r = reduce_state(*this, true);
  reset_errors();
  return r.ke;
}

void DevSystem::check_finite(uint64_t step) {
  reset_errors();
  reduce_state(*this, false);
  DScalars hs;
  CK(cudaMemcpy(&hs, scal.p, sizeof(DScalars), cudaMemcpyDeviceToHost));
  if (hs.failed) {
    hs.err_step = static_cast<long long>(step);
    CK(cudaMemcpy(scal.p, &hs, sizeof(DScalars), cudaMemcpyHostToDevice));
    raise_if_failed("check_finite");
  }
}

// |v|max, |a|max and kinetic energy over the owned particles; a non-finite
// owned particle fails with the check_finite message for `step` (check >= 0).
void DevSystem::reduce_owned(bool want_ke, long long check_step, double out[3]) {
  reset_errors();
  const Reduced r = reduce_state(*this, want_ke);
  out[0] = r.vmax;
  out[1] = r.amax;
  out[2] = r.ke;
  if (check_step < 0) {
    reset_errors();
    return;
  }
  DScalars hs;
  CK(cudaMemcpy(&hs, scal.p, sizeof(DScalars), cudaMemcpyDeviceToHost));
  if (hs.failed) {
    hs.err_step = check_step;
    CK(cudaMemcpy(scal.p, &hs, sizeof(DScalars), cudaMemcpyHostToDevice));
    raise_if_failed("check_finite");
  }
}

}  // namespace tlsph_cuda
