"""Python mirror of the reference operator API over the B200 C ABI (libtlsph_cuda.so).

Every call goes through include/tlsph/tlsph_dev.h into the sm_100a kernels;
there is no CPU fallback: importing this module on a machine without the
built library raises, and every compute call on a machine without a GPU
fails with the CUDA error mapped to TLSPH_ERR_INTERNAL.

Names and argument meaning follow the reference C++ operator API
(proj/src/tlsph/{neighbors,damping,integrator}.hpp):

    sys = DeviceSystem(r0, V0, rho0, h, constrained)   # build_cell_grid + block_decompose
                                                      # + build_reference_neighborhoods
    sys.correction_matrices()                          # compute_correction_matrices
    sys.damping_sweep("particle_split", eta_tilde, dt) # strang_damping_sweep
    sys.verlet_step(material, dt)                      # verlet_step
    ...

Arrays are numpy float64 in reference particle order.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_PKG, "lib")
CUDA_LIB = os.environ.get("TLSPH_CUDA_LIB", os.path.join(LIB_DIR, "libtlsph_cuda.so"))

STATUS = {0: "ok", 1: "invalid-argument", 2: "parse-error", 3: "degenerate-geometry", 4: "inverted-element",
          5: "numerical-failure", 6: "io-error", 7: "internal-error"}
FIELDS = {"r0": 0, "r": 1, "v": 2, "a": 3, "F": 4, "dFdt": 5, "B0": 6, "V0": 7, "m": 8, "rho0": 9, "rho": 10,
          "body": 11, "constrained": 12}
_VEC = {"r0", "r", "v", "a", "body"}
_MAT = {"F", "dFdt", "B0"}
SCHEMES = {"explicit": 0, "particle_split": 1, "pairwise_split": 2}
COLUMN_FIELDS = {"velocity": 0, "stress": 1}  # tlsph_dev_column_field


class TlsphError(RuntimeError):
    """A non-OK tlsph_status with the library's message (reference capi.cpp:26-42 semantics)."""

    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status
        self.kind = STATUS.get(status, str(status))
        self.message = message


class Material(C.Structure):
    """tlsph_dev_material (material.hpp:16-27)."""

    _fields_ = [("model", C.c_int), ("lambda_", C.c_double), ("mu", C.c_double), ("K", C.c_double),
                ("G", C.c_double), ("E", C.c_double), ("nu", C.c_double), ("rho0", C.c_double), ("c", C.c_double)]

    @classmethod
    def from_young_poisson(cls, E, nu, rho0, model="neo_hookean"):
        """material_from_young_poisson (material.cpp:10-30)."""
        if not E > 0.0:
            raise TlsphError(1, f"Young's modulus must be positive, got {E}")
        if not (0.0 <= nu < 0.5):
            raise TlsphError(1, f"Poisson ratio must lie in [0, 0.5), got {nu}")
        if not rho0 > 0.0:
            raise TlsphError(1, f"reference density must be positive, got {rho0}")
        mu = E / (2.0 * (1.0 + nu))
        lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
        K = lam + 2.0 * mu / 3.0
        c = float(np.sqrt(K / rho0))
        return cls(1 if model == "neo_hookean" else 0, lam, mu, K, mu, E, nu, rho0, c)


class LoopParams(C.Structure):
    _fields_ = [("material", Material), ("h", C.c_double), ("eta", C.c_double), ("alpha", C.c_double),
                ("scheme", C.c_int), ("seed", C.c_uint64), ("end_time", C.c_double), ("max_steps", C.c_uint64),
                ("fixed_dt", C.c_double), ("elastic", C.c_int), ("ke_stop", C.c_int), ("ke_ratio", C.c_double),
                ("probe_index", C.c_int64), ("output_interval", C.c_double), ("probe_out", C.POINTER(C.c_double)),
                ("probe_capacity", C.c_size_t), ("pause_on_mark", C.c_int), ("resume", C.c_int)]


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_int)


class GroupComm(C.Structure):
    """tlsph_group_comm: the caller's collectives for a tlsph_dev_group (tlsph_dev.h)."""
    _fields_ = [("ctx", C.c_void_p), ("rank", C.c_int), ("size", C.c_int), ("allgather", ALLGATHER_FN),
                ("allreduce_f64", ALLREDUCE_FN)]


class LoopResult(C.Structure):
    _fields_ = [("steps", C.c_uint64), ("damped_steps", C.c_uint64), ("t", C.c_double), ("last_dt", C.c_double),
                ("elastic_seconds", C.c_double), ("damping_seconds", C.c_double), ("total_seconds", C.c_double),
                ("peak_ke", C.c_double), ("final_ke", C.c_double), ("stopped_on_ke", C.c_int),
                ("probe_samples", C.c_size_t), ("paused", C.c_int), ("kernel_launches", C.c_uint64)]


_lib = None


def lib():
    """Loads libtlsph_cuda.so; raises if it was not built (no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(CUDA_LIB):
        raise ImportError(f"{CUDA_LIB} is missing: run __graft_entry__.build() (make -C paper_2103_08932_b200/csrc)")
    L = C.CDLL(CUDA_LIB)
    P, D, I, S = C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_size_t
    L.tlsph_dev_last_error.restype = C.c_char_p
    L.tlsph_dev_device_count.restype = C.c_int
    L.tlsph_dev_select_device.argtypes = [C.c_int]
    L.tlsph_dev_create.argtypes = [I, S, D, D, D, C.POINTER(C.c_uint8), C.c_double, C.POINTER(P)]
    L.tlsph_dev_create_with_csr.argtypes = [I, S, D, D, D, C.POINTER(C.c_uint8), C.c_double,
                                            C.POINTER(C.c_int64), C.POINTER(C.c_int32), D, D, D, D, C.POINTER(P)]
    L.tlsph_dev_create_in_grid.argtypes = [I, S, D, D, D, C.POINTER(C.c_uint8), C.c_double, D, C.POINTER(I),
                                           C.POINTER(P)]
    L.tlsph_dev_set_task_range.argtypes = [P, I, I]
    L.tlsph_dev_damping_phase.argtypes = [P, I, C.c_double, C.c_double, I, I]
    L.tlsph_dev_link_peer.argtypes = [P, I, P]
    L.tlsph_dev_column_count.argtypes = [P, I]
    L.tlsph_dev_column_count.restype = C.c_int64
    L.tlsph_dev_pack_column.argtypes = [P, I, C.c_void_p]
    L.tlsph_dev_unpack_column.argtypes = [P, I, C.c_void_p]
    L.tlsph_dev_column_width.argtypes = [P, I]
    L.tlsph_dev_pack_column_field.argtypes = [P, I, I, C.c_void_p]
    L.tlsph_dev_unpack_column_field.argtypes = [P, I, I, C.c_void_p]
    L.tlsph_dev_verlet_pass.argtypes = [P, C.POINTER(Material), C.c_double, I]
    L.tlsph_dev_reduce_state.argtypes = [P, I, C.c_int64, D]
    L.tlsph_dev_destroy.argtypes = [P]
    L.tlsph_dev_size.argtypes = [P]
    L.tlsph_dev_size.restype = S
    L.tlsph_dev_dim.argtypes = [P]
    L.tlsph_dev_slot_count.argtypes = [P]
    L.tlsph_dev_slot_count.restype = C.c_int64
    L.tlsph_dev_set_field.argtypes = [P, I, D]
    L.tlsph_dev_get_field.argtypes = [P, I, D]
    L.tlsph_dev_set_reduction.argtypes = [P, I]
    L.tlsph_dev_sweep_linked.argtypes = [C.POINTER(P), I, I, C.c_double, C.c_double, I]
    L.tlsph_dev_set_sweep_tiling.argtypes = [P, I]
    L.tlsph_dev_set_sweep_blocking.argtypes = [P, I, I]
    L.tlsph_dev_set_resort.argtypes = [P, I]
    L.tlsph_dev_last_run_steps.argtypes = [P]
    L.tlsph_dev_last_run_steps.restype = C.c_int64
    L.tlsph_dev_last_run_time.argtypes = [P]
    L.tlsph_dev_last_run_time.restype = C.c_double
    L.tlsph_dev_current_cells.argtypes = [P, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
    L.tlsph_dev_ipc_size.argtypes = []
    L.tlsph_dev_ipc_size.restype = S
    L.tlsph_dev_ipc_export.argtypes = [P, C.c_void_p]
    L.tlsph_dev_link_peer_ipc.argtypes = [P, I, C.c_char_p, C.POINTER(C.c_int64)]
    L.tlsph_dev_sweep_phase_ipc.argtypes = [P, I, C.c_double, C.c_double, I, I]
    L.tlsph_dev_synchronize.argtypes = [P]
    L.tlsph_dev_push_halo_ipc.argtypes = [P, I]
    L.tlsph_dev_wait_halo_ipc.argtypes = [P, I]
    L.tlsph_dev_mark_ipc.argtypes = [P]
    L.tlsph_dev_wait_mark_ipc.argtypes = [P]
    L.tlsph_dev_wait_phase_ipc.argtypes = [P, I]
    L.tlsph_dev_timer_start.argtypes = [P]
    L.tlsph_dev_timer_stop.argtypes = [P]
    L.tlsph_dev_timer_stop.restype = C.c_double
    L.tlsph_dev_grid_info.argtypes = [P, C.POINTER(I), D, D, C.POINTER(C.c_int64)]
    L.tlsph_dev_grid_cells.argtypes = [P, C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
    L.tlsph_dev_get_neighborhood.argtypes = [P, C.POINTER(C.c_int64), C.POINTER(C.c_int32), D, D, D, D]
    for name in ("tlsph_dev_correction_matrices", "tlsph_dev_deformation_rate", "tlsph_dev_update_density",
                 "tlsph_dev_apply_constraints"):
        getattr(L, name).argtypes = [P]
    L.tlsph_dev_momentum_rhs.argtypes = [P, C.POINTER(Material)]
    L.tlsph_dev_verlet_step.argtypes = [P, C.POINTER(Material), C.c_double]
    L.tlsph_dev_stable_dt.argtypes = [P, C.POINTER(Material), C.c_double, D]
    L.tlsph_dev_kinetic_energy.argtypes = [P, D]
    L.tlsph_dev_check_finite.argtypes = [P, C.c_uint64]
    L.tlsph_dev_damping_sweep.argtypes = [P, I, C.c_double, C.c_double]
    L.tlsph_dev_damping_sweeps.argtypes = [P, I, C.c_double, C.c_double, I]
    L.tlsph_dev_particle_split_update.argtypes = [P, S, C.c_double, C.c_double]
    L.tlsph_dev_pairwise_split_update.argtypes = [P, S, C.c_int64, C.c_double, C.c_double]
    L.tlsph_dev_explicit_damping_accel.argtypes = [P, C.c_double, D]
    L.tlsph_dev_run.argtypes = [P, C.POINTER(LoopParams), C.POINTER(LoopResult)]
    L.tlsph_dev_group_create.argtypes = [P, C.POINTER(GroupComm), C.POINTER(C.c_void_p)]
    L.tlsph_dev_group_sweep.argtypes = [P, I, C.c_double, C.c_double, I]
    L.tlsph_dev_group_run.argtypes = [P, C.POINTER(LoopParams), C.POINTER(LoopResult)]
    L.tlsph_dev_group_destroy.argtypes = [P]
    L.tlsph_dev_group_destroy.restype = None
    L.tlsph_group_last_error.restype = C.c_char_p
    L.tlsph_group_plan.argtypes = [C.POINTER(C.c_int64), I, I, I, C.POINTER(C.c_int)]
    L.tlsph_group_step_dt.argtypes = [C.POINTER(LoopParams), I, C.c_double, C.c_double]
    L.tlsph_group_step_dt.restype = C.c_double
    L.tlsph_group_comm_selftest.argtypes = [C.POINTER(GroupComm)]
    L.tlsph_random_uniforms.argtypes = [C.c_uint64, S, D]
    L.tlsph_random_choice.argtypes = [C.c_double, C.c_double, C.c_uint64, S, D]
    L.tlsph_dev_last_elapsed.argtypes = [P]
    L.tlsph_dev_last_elapsed.restype = C.c_double
    L.tlsph_dev_selftest_division.argtypes = [C.c_int64, C.c_uint64, C.POINTER(C.c_uint64)]
    _lib = L
    return L


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def sweep_linked(systems, scheme, eta_tilde, dt, count=1):
    """tlsph_dev_sweep_linked: `count` sweeps over peer-linked slabs (left to right) with the
    per-phase ordering kept on the devices; returns the device time of the call (seconds)."""
    arr = (C.c_void_p * len(systems))(*[d._h.value for d in systems])
    _check(lib().tlsph_dev_sweep_linked(arr, len(systems), SCHEMES[scheme], float(eta_tilde), float(dt), int(count)))
    return float(lib().tlsph_dev_last_elapsed(systems[0]._h))


def _check(status):
    if status != 0:
        raise TlsphError(status, lib().tlsph_dev_last_error().decode())


def device_count() -> int:
    return int(lib().tlsph_dev_device_count())


def select_device(ordinal: int) -> None:
    """Device for handles created afterwards (one process per GPU: LOCAL_RANK)."""
    _check(lib().tlsph_dev_select_device(ordinal))


def selftest_division(n=1 << 26, seed=1):
    """Mismatches of the corrected quotient against IEEE division on the device (expected 0)."""
    out = C.c_uint64()
    _check(lib().tlsph_dev_selftest_division(n, seed, C.byref(out)))
    return int(out.value)


def random_uniforms(seed, n):
    out = np.empty(n)
    _check(lib().tlsph_random_uniforms(seed, n, _dp(out)))
    return out


def random_choice(eta, alpha, seed, n):
    out = np.empty(n)
    _check(lib().tlsph_random_choice(eta, alpha, seed, n, _dp(out)))
    return out


class DeviceSystem:
    """Device-resident ParticleSystem<D> + CellGrid + ReferenceNeighborhood (sorted SoA on the GPU)."""

    def __init__(self, r0, V0, rho0, h, constrained=None, csr=None, grid=None):
        """grid=(origin, dims): bin into that (global) cell grid instead of the
        bounding box of r0 -- one x-slab of a decomposed body (tlsph_dev_create_in_grid)."""
        r0 = np.ascontiguousarray(r0, dtype=np.float64)
        self.n, self.dim = r0.shape
        V0 = np.ascontiguousarray(np.broadcast_to(np.asarray(V0, dtype=np.float64), (self.n,)))
        rho0 = np.ascontiguousarray(np.broadcast_to(np.asarray(rho0, dtype=np.float64), (self.n,)))
        cons = None if constrained is None else np.ascontiguousarray(constrained, dtype=np.uint8)
        cons_p = cons.ctypes.data_as(C.POINTER(C.c_uint8)) if cons is not None else None
        self.h = float(h)
        self._h = C.c_void_p()
        if grid is not None:
            origin = np.zeros(3)
            origin[: self.dim] = np.asarray(grid[0], dtype=np.float64)[: self.dim]
            dims = (C.c_int * 3)(*[int(x) for x in list(grid[1])[: self.dim]] + [1] * (3 - self.dim))
            _check(lib().tlsph_dev_create_in_grid(self.dim, self.n, _dp(r0), _dp(V0), _dp(rho0), cons_p, self.h,
                                                  _dp(origin), dims, C.byref(self._h)))
        elif csr is None:
            _check(lib().tlsph_dev_create(self.dim, self.n, _dp(r0), _dp(V0), _dp(rho0), cons_p, self.h,
                                          C.byref(self._h)))
        else:
            off = np.ascontiguousarray(csr["offsets"], dtype=np.int64)
            nb = np.ascontiguousarray(csr["neighbor"], dtype=np.int32)
            arrs = [np.ascontiguousarray(csr[k], dtype=np.float64) for k in ("r0_len", "e0", "dwdr0", "pair_factor")]
            _check(lib().tlsph_dev_create_with_csr(
                self.dim, self.n, _dp(r0), _dp(V0), _dp(rho0), cons_p, self.h,
                off.ctypes.data_as(C.POINTER(C.c_int64)), nb.ctypes.data_as(C.POINTER(C.c_int32)),
                *[_dp(a) for a in arrs], C.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().tlsph_dev_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def slot_count(self):
        return int(lib().tlsph_dev_slot_count(self._h))

    def set_reduction(self, mode):
        _check(lib().tlsph_dev_set_reduction(self._h, {"fast": 0, "ordered": 1}[mode]))

    def set_resort(self, on=True):
        """BASELINE cfg4's per-step re-sort: the device loop rebuilds the current-position cell list."""
        _check(lib().tlsph_dev_set_resort(self._h, 1 if on else 0))

    def current_cells(self):
        """(cell_start, reference ids in current-cell order) of the last re-sort."""
        g = self.grid()
        cs = np.zeros(len(g["cell_start"]), dtype=np.int64)
        order = np.zeros(self.n, dtype=np.int32)
        _check(lib().tlsph_dev_current_cells(self._h, cs.ctypes.data_as(C.POINTER(C.c_int64)),
                                             order.ctypes.data_as(C.POINTER(C.c_int32))))
        return cs, order

    def set_sweep_tiling(self, mode):
        """FAST sweep slot-block placement: "auto", "staged" (shared memory) or "streamed" (L2)."""
        _check(lib().tlsph_dev_set_sweep_tiling(self._h, {"auto": 0, "staged": 1, "streamed": 2}[mode]))

    def set_sweep_blocking(self, columns=-1, phases=0):
        """Temporal blocking of the sweep's phase schedule over x-column chunks (-1: automatic,
        0: off); results are bitwise those of the phase-by-phase order."""
        _check(lib().tlsph_dev_set_sweep_blocking(self._h, int(columns), int(phases)))

    # ---- fields
    def _shape(self, name):
        if name in _VEC:
            return (self.n, self.dim)
        if name in _MAT:
            return (self.n, self.dim, self.dim)
        return (self.n,)

    def get(self, name, out=None):
        """Field in reference order; `out` (e.g. a pinned host array) receives it when given."""
        if out is None:
            out = np.empty(self._shape(name))
        elif out.shape != self._shape(name) or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError(f"out must be a C-contiguous float64 array of shape {self._shape(name)}")
        _check(lib().tlsph_dev_get_field(self._h, FIELDS[name], _dp(out)))
        return out

    def set(self, name, value):
        arr = np.ascontiguousarray(np.broadcast_to(np.asarray(value, dtype=np.float64), self._shape(name)))
        _check(lib().tlsph_dev_set_field(self._h, FIELDS[name], _dp(arr)))

    # ---- cell grid / neighbourhood (reference layout)
    def grid(self):
        dims = (C.c_int * 3)()
        origin = (C.c_double * 3)()
        cs = C.c_double()
        nc = C.c_int64()
        _check(lib().tlsph_dev_grid_info(self._h, dims, origin, C.byref(cs), C.byref(nc)))
        cell_of = np.empty(self.n, dtype=np.int32)
        cell_start = np.empty(nc.value + 1, dtype=np.int64)
        cell_particles = np.empty(self.n, dtype=np.int32)
        _check(lib().tlsph_dev_grid_cells(self._h, cell_of.ctypes.data_as(C.POINTER(C.c_int32)),
                                          cell_start.ctypes.data_as(C.POINTER(C.c_int64)),
                                          cell_particles.ctypes.data_as(C.POINTER(C.c_int32))))
        return {"dims": list(dims)[: self.dim], "origin": list(origin)[: self.dim], "cell_size": cs.value,
                "cell_of": cell_of, "cell_start": cell_start, "cell_particles": cell_particles}

    def blocks(self):
        """block_decompose (neighbors.cpp:61-77): colour of a cell = sum_d (c_d mod 3) 3^d, ascending cells."""
        g = self.grid()
        dims = g["dims"]
        ncell = int(np.prod(dims))
        lin = np.arange(ncell)
        colour = np.zeros(ncell, dtype=np.int64)
        stride = 1
        rem = lin.copy()
        for d in range(self.dim):
            colour += (rem % dims[d]) % 3 * stride
            rem //= dims[d]
            stride *= 3
        return [lin[colour == b].tolist() for b in range(3 ** self.dim)]

    def row_offsets(self):
        """Reference-order CSR row offsets only (no slot arrays transferred)."""
        off = np.empty(self.n + 1, dtype=np.int64)
        _check(lib().tlsph_dev_get_neighborhood(self._h, off.ctypes.data_as(C.POINTER(C.c_int64)), None, None, None,
                                                None, None))
        return off

    def neighborhood(self, fields=None):
        """ReferenceNeighborhood arrays; `fields` (names) limits which are copied out."""
        want = set(fields) if fields is not None else {"offsets", "neighbor", "r0_len", "e0", "dwdr0", "pair_factor"}
        S = self.slot_count
        off = np.empty(self.n + 1, dtype=np.int64)
        nb = np.empty(S if "neighbor" in want else 0, dtype=np.int32)
        ln = np.empty(S if "r0_len" in want else 0)
        e0 = np.empty((S if "e0" in want else 0, self.dim))
        dw = np.empty(S if "dwdr0" in want else 0)
        pf = np.empty(S if "pair_factor" in want else 0)

        def ptr(a, name, t=None):
            if name not in want:
                return None
            return a.ctypes.data_as(C.POINTER(t)) if t is not None else _dp(a)

        _check(lib().tlsph_dev_get_neighborhood(self._h, off.ctypes.data_as(C.POINTER(C.c_int64)), ptr(nb, "neighbor", C.c_int32),
                        ptr(ln, "r0_len"), ptr(e0, "e0"), ptr(dw, "dwdr0"), ptr(pf, "pair_factor")))
        out = {"offsets": off, "neighbor": nb, "r0_len": ln, "e0": e0, "dwdr0": dw, "pair_factor": pf}
        return {k: v for k, v in out.items() if k in want or k == "offsets"}

    # ---- operators
    def correction_matrices(self):
        _check(lib().tlsph_dev_correction_matrices(self._h))

    def deformation_rate(self):
        _check(lib().tlsph_dev_deformation_rate(self._h))

    def update_density(self):
        _check(lib().tlsph_dev_update_density(self._h))

    def momentum_rhs(self, material):
        _check(lib().tlsph_dev_momentum_rhs(self._h, C.byref(material)))

    def verlet_step(self, material, dt):
        _check(lib().tlsph_dev_verlet_step(self._h, C.byref(material), dt))

    def apply_constraints(self):
        _check(lib().tlsph_dev_apply_constraints(self._h))

    def stable_dt(self, material, h=None):
        out = C.c_double()
        _check(lib().tlsph_dev_stable_dt(self._h, C.byref(material), self.h if h is None else h, C.byref(out)))
        return out.value

    def kinetic_energy(self):
        out = C.c_double()
        _check(lib().tlsph_dev_kinetic_energy(self._h, C.byref(out)))
        return out.value

    def check_finite(self, step):
        _check(lib().tlsph_dev_check_finite(self._h, step))

    def damping_sweep(self, scheme, eta_tilde, dt, count=1):
        if count == 1:
            _check(lib().tlsph_dev_damping_sweep(self._h, SCHEMES[scheme], eta_tilde, dt))
        else:
            _check(lib().tlsph_dev_damping_sweeps(self._h, SCHEMES[scheme], eta_tilde, dt, count))
        return float(lib().tlsph_dev_last_elapsed(self._h))

    # ---- x-slab decomposition (paper_2103_08932_b200/slabs.py)
    def set_task_range(self, x0, x1):
        _check(lib().tlsph_dev_set_task_range(self._h, int(x0), int(x1)))

    def damping_phase(self, scheme, eta_tilde, dt, pass_, index):
        _check(lib().tlsph_dev_damping_phase(self._h, SCHEMES[scheme], float(eta_tilde), float(dt), int(pass_),
                                             int(index)))

    # ---- cross-process linking (one process per GPU; slabs.IpcSlabSweep)
    def ipc_export(self):
        """This slab's velocity arrays and phase events as CUDA IPC handles (opaque bytes)."""
        buf = C.create_string_buffer(int(lib().tlsph_dev_ipc_size()))
        _check(lib().tlsph_dev_ipc_export(self._h, C.cast(buf, C.c_void_p)))
        return buf.raw

    def link_peer_ipc(self, side, blob, peer_cell_start):
        """Fused exchange with a slab of another process: its export and its cell table."""
        cs = np.ascontiguousarray(peer_cell_start, dtype=np.int64)
        _check(lib().tlsph_dev_link_peer_ipc(self._h, int(side), bytes(blob), cs.ctypes.data_as(C.POINTER(C.c_int64))))

    def sweep_phase_ipc(self, scheme, eta_tilde, dt, q, wait_q):
        """Enqueue colour phase q after the linked neighbours' phase wait_q (-1: no wait); asynchronous."""
        _check(lib().tlsph_dev_sweep_phase_ipc(self._h, SCHEMES[scheme], float(eta_tilde), float(dt), int(q),
                                               int(wait_q)))

    def synchronize(self):
        _check(lib().tlsph_dev_synchronize(self._h))

    def push_halo_ipc(self, field):
        """Store this slab's owned boundary columns of `field` into the linked neighbours (async)."""
        _check(lib().tlsph_dev_push_halo_ipc(self._h, COLUMN_FIELDS[field]))

    def wait_halo_ipc(self, field):
        """This slab's stream waits on the neighbours' halo pushes of `field` (async)."""
        _check(lib().tlsph_dev_wait_halo_ipc(self._h, COLUMN_FIELDS[field]))

    def mark_ipc(self):
        """Records this slab's mark event after all work enqueued so far (async)."""
        _check(lib().tlsph_dev_mark_ipc(self._h))

    def wait_mark_ipc(self):
        """This slab's stream waits on the neighbours' mark events (async)."""
        _check(lib().tlsph_dev_wait_mark_ipc(self._h))

    def wait_phase_ipc(self, q):
        """This slab's stream waits on the neighbours' colour-phase-q events (async)."""
        _check(lib().tlsph_dev_wait_phase_ipc(self._h, int(q)))

    def timer_start(self):
        """Start a device-time span on this system's stream (timer_stop returns its seconds)."""
        _check(lib().tlsph_dev_timer_start(self._h))

    def timer_stop(self):
        t = float(lib().tlsph_dev_timer_stop(self._h))
        if t < 0:
            raise TlsphError(1, lib().tlsph_dev_last_error().decode())
        return t

    def link_peer(self, side, peer):
        """Fused exchange: this slab's phases also store the shared columns into `peer` (0 left, 1 right)."""
        _check(lib().tlsph_dev_link_peer(self._h, int(side), peer._h))

    def column_count(self, x):
        c = int(lib().tlsph_dev_column_count(self._h, int(x)))
        if c < 0:
            raise TlsphError(1, lib().tlsph_dev_last_error().decode())
        return c

    def column_width(self, field="velocity"):
        """Doubles per particle of a column field ("velocity": D, "stress": D*D + 1)."""
        w = int(lib().tlsph_dev_column_width(self._h, COLUMN_FIELDS[field]))
        if w < 0:
            raise TlsphError(1, lib().tlsph_dev_last_error().decode())
        return w

    def pack_column(self, x, device_ptr, field="velocity"):
        """Field of cell column x into the device buffer at device_ptr (width x count doubles)."""
        _check(lib().tlsph_dev_pack_column_field(self._h, COLUMN_FIELDS[field], int(x), C.c_void_p(int(device_ptr))))

    def unpack_column(self, x, device_ptr, field="velocity"):
        _check(lib().tlsph_dev_unpack_column_field(self._h, COLUMN_FIELDS[field], int(x),
                                                   C.c_void_p(int(device_ptr))))

    def verlet_pass(self, material, dt, pass_):
        """One pass of verlet_step: 0 = A (stress record), 1 = B (momentum + kick), 2 = C (dF/dt)."""
        _check(lib().tlsph_dev_verlet_pass(self._h, C.byref(material), float(dt), int(pass_)))

    def reduce_state(self, want_ke=False, check_step=-1):
        """(|v|max, |a|max, kinetic energy) over the owned particles; check_step >= 0 also runs
        check_finite for that step."""
        out = np.zeros(3)
        _check(lib().tlsph_dev_reduce_state(self._h, 1 if want_ke else 0, int(check_step), _dp(out)))
        return float(out[0]), float(out[1]), float(out[2])

    def particle_split_update(self, i, eta, dt_half):
        _check(lib().tlsph_dev_particle_split_update(self._h, i, eta, dt_half))

    def pairwise_split_update(self, i, slot, eta, dt_half):
        _check(lib().tlsph_dev_pairwise_split_update(self._h, i, slot, eta, dt_half))

    def explicit_damping_accel(self, eta):
        out = np.empty((self.n, self.dim))
        _check(lib().tlsph_dev_explicit_damping_accel(self._h, eta, _dp(out)))
        return out

    def run(self, material, *, eta, alpha, scheme="particle_split", steps=0, end_time=0.0, fixed_dt=0.0,
            elastic=True, seed=0, ke_stop=False, ke_ratio=1e-8, resume=False):
        """Device-resident loop of runner.cpp:341-391 (state must be prepared as :306-312 does).
        resume=True continues the previous loop (same eta~ stream, t and step count; `steps` is the
        cumulative cap); the returned times are then cumulative too."""
        p = LoopParams(material, self.h, eta, alpha, SCHEMES[scheme], seed, end_time, steps, fixed_dt,
                       1 if elastic else 0, 1 if ke_stop else 0, ke_ratio, -1, 0.0, None, 0, 0,
                       1 if resume else 0)
        r = LoopResult()
        _check(lib().tlsph_dev_run(self._h, C.byref(p), C.byref(r)))
        return {"steps": r.steps, "damped": r.damped_steps, "t": r.t, "last_dt": r.last_dt,
                "elastic_s": r.elastic_seconds, "damping_s": r.damping_seconds, "total_s": r.total_seconds,
                "peak_ke": r.peak_ke, "final_ke": r.final_ke, "stopped_on_ke": bool(r.stopped_on_ke),
                "kernel_launches": int(r.kernel_launches)}

    def last_run(self):
        """(completed steps, t) of the last run, also when it stopped on an error."""
        return int(lib().tlsph_dev_last_run_steps(self._h)), float(lib().tlsph_dev_last_run_time(self._h))

    def prepare(self, material):
        """runner.cpp:306-312: B0, constraints, initial momentum RHS and deformation rate."""
        self.correction_matrices()
        self.apply_constraints()
        self.momentum_rhs(material)
        self.deformation_rate()
