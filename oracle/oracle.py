"""TEST INFRASTRUCTURE ONLY — ctypes binding of the CPU oracle (oracle/_build/liboracle.so).

The oracle restates the reference's hot path on the CPU (see tlsph_oracle.hpp).
Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
reference) may import this module, and only as the checker or the CPU
baseline. The product package never imports it.

Arrays are numpy float64 in reference particle order: vectors (n, D),
matrices (n, D, D) row-major.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

FIELDS = {"r0": 0, "r": 1, "v": 2, "a": 3, "F": 4, "dFdt": 5, "B0": 6, "V0": 7, "m": 8,
          "rho0": 9, "rho": 10, "body": 11, "constrained": 12}
_VEC = {"r0", "r", "v", "a", "body"}
_MAT = {"F", "dFdt", "B0"}

SCHEMES = {"explicit": 0, "particle_split": 1, "pairwise_split": 2}

ERROR_KINDS = {1: "invalid-argument", 2: "parse-error", 3: "degenerate-geometry",
               4: "inverted-element", 5: "numerical-failure", 6: "io-error", 7: "internal-error"}


class OracleError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{ERROR_KINDS.get(status, status)}: {message}")
        self.status = status
        self.kind = ERROR_KINDS.get(status, str(status))
        self.message = message


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        D = C.POINTER(C.c_double)
        I = C.c_int
        L.orc_last_error.restype = C.c_char_p
        L.orc_create.argtypes = [I, C.c_size_t, D, D, D, C.POINTER(C.c_ubyte), C.c_double, I, C.POINTER(P)]
        L.orc_destroy.argtypes = [P]
        L.orc_size.argtypes = [P]
        L.orc_size.restype = C.c_size_t
        L.orc_set_field.argtypes = [P, I, D]
        L.orc_get_field.argtypes = [P, I, D]
        L.orc_set_material.argtypes = [P, C.c_double, C.c_double, C.c_double, I]
        L.orc_material.argtypes = [C.c_double, C.c_double, C.c_double, I, D]
        L.orc_grid_info.argtypes = [P, C.POINTER(I), D, D, C.POINTER(C.c_longlong)]
        L.orc_grid_cells.argtypes = [P, C.POINTER(I), C.POINTER(C.c_longlong), C.POINTER(I)]
        L.orc_blocks.argtypes = [P, C.POINTER(C.c_longlong), C.POINTER(I)]
        L.orc_slot_count.argtypes = [P]
        L.orc_slot_count.restype = C.c_longlong
        L.orc_get_neighborhood.argtypes = [P, C.POINTER(C.c_longlong), C.POINTER(I), D, D, D, D]
        L.orc_set_neighborhood.argtypes = [P, C.POINTER(C.c_longlong), C.POINTER(I), D, D, D, D]
        for name in ("orc_correction_matrices", "orc_deformation_rate", "orc_update_density",
                     "orc_momentum_rhs", "orc_prepare"):
            getattr(L, name).argtypes = [P, I]
        L.orc_verlet_step.argtypes = [P, C.c_double, I]
        L.orc_apply_constraints.argtypes = [P]
        L.orc_stable_dt.argtypes = [P, C.c_double, D]
        L.orc_kinetic_energy.argtypes = [P, D]
        L.orc_check_finite.argtypes = [P, C.c_ulonglong]
        L.orc_damping_sweep.argtypes = [P, I, C.c_double, C.c_double, I]
        L.orc_particle_split_update.argtypes = [P, C.c_size_t, C.c_double, C.c_double]
        L.orc_pairwise_split_update.argtypes = [P, C.c_size_t, C.c_longlong, C.c_double, C.c_double]
        L.orc_explicit_damping_accel.argtypes = [P, C.c_double, D, I]
        L.orc_grad_mag.argtypes = [C.c_double, I, C.c_double, D]
        L.orc_kernel_value.argtypes = [C.c_double, I, C.c_double, D]
        L.orc_random_uniforms.argtypes = [C.c_ulonglong, C.c_size_t, D]
        L.orc_random_choice.argtypes = [C.c_double, C.c_double, C.c_ulonglong, C.c_size_t, D]
        L.orc_viscous_bounds.argtypes = [C.c_double, C.c_double, I, D]
        L.orc_artificial_viscosity.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, D]
        L.orc_second_pk.argtypes = [I, D, C.c_double, C.c_double, C.c_double, I, D]
        L.orc_box_lattice.argtypes = [I, D, D, C.c_double, D]
        L.orc_box_lattice.restype = C.c_longlong
        L.orc_run.argtypes = [P, D, D]
        L.orc_run_probed.argtypes = [P, D, D, D, C.c_longlong, C.POINTER(C.c_longlong)]
        L.orc_set_contact.argtypes = [P, D, D, C.c_double]
        L.orc_last_run.argtypes = [P, D]
        L.orc_openmp_threads.restype = C.c_int
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


def _check(status):
    if status != 0:
        raise OracleError(status, lib().orc_last_error().decode())


def openmp_threads() -> int:
    return int(lib().orc_openmp_threads())


class OracleSystem:
    """A ParticleSystem<D> + CellGrid + blocks + ReferenceNeighborhood held by the oracle."""

    def __init__(self, r0, V0, rho0, h, constrained=None, build=True):
        r0 = np.ascontiguousarray(r0, dtype=np.float64)
        self.n, self.dim = r0.shape
        V0 = np.ascontiguousarray(np.broadcast_to(np.asarray(V0, dtype=np.float64), (self.n,)))
        rho0 = np.ascontiguousarray(np.broadcast_to(np.asarray(rho0, dtype=np.float64), (self.n,)))
        cons = None
        if constrained is not None:
            cons = np.ascontiguousarray(constrained, dtype=np.uint8)
        self.h = float(h)
        self._h = C.c_void_p()
        _check(lib().orc_create(self.dim, self.n, _dp(r0), _dp(V0), _dp(rho0),
                                cons.ctypes.data_as(C.POINTER(C.c_ubyte)) if cons is not None else None,
                                self.h, 1 if build else 0, C.byref(self._h)))

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None and self._h.value:
                lib().orc_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass

    # ---- fields
    def _shape(self, name):
        if name in _VEC:
            return (self.n, self.dim)
        if name in _MAT:
            return (self.n, self.dim, self.dim)
        return (self.n,)

    def get(self, name):
        out = np.empty(self._shape(name), dtype=np.float64)
        _check(lib().orc_get_field(self._h, FIELDS[name], _dp(out)))
        return out

    def set(self, name, value):
        arr = np.ascontiguousarray(np.broadcast_to(np.asarray(value, dtype=np.float64), self._shape(name)))
        _check(lib().orc_set_field(self._h, FIELDS[name], _dp(arr)))

    def set_material(self, E, nu, rho0, model="neo_hookean"):
        _check(lib().orc_set_material(self._h, E, nu, rho0, 1 if model == "neo_hookean" else 0))

    # ---- grid / blocks / neighbourhood
    def grid(self):
        dims = (C.c_int * 3)()
        origin = (C.c_double * 3)()
        cs = C.c_double()
        nc = C.c_longlong()
        _check(lib().orc_grid_info(self._h, dims, origin, C.byref(cs), C.byref(nc)))
        ncell = nc.value
        cell_of = np.empty(self.n, dtype=np.int32)
        cell_start = np.empty(ncell + 1, dtype=np.int64)
        cell_particles = np.empty(self.n, dtype=np.int32)
        _check(lib().orc_grid_cells(self._h, cell_of.ctypes.data_as(C.POINTER(C.c_int)),
                                    cell_start.ctypes.data_as(C.POINTER(C.c_longlong)),
                                    cell_particles.ctypes.data_as(C.POINTER(C.c_int))))
        return {"dims": list(dims)[: self.dim], "origin": list(origin)[: self.dim], "cell_size": cs.value,
                "cell_of": cell_of, "cell_start": cell_start, "cell_particles": cell_particles}

    def blocks(self):
        g = self.grid()
        ncell = len(g["cell_start"]) - 1
        nb = 9 if self.dim == 2 else 27
        bs = np.empty(nb + 1, dtype=np.int64)
        bc = np.empty(ncell, dtype=np.int32)
        _check(lib().orc_blocks(self._h, bs.ctypes.data_as(C.POINTER(C.c_longlong)), bc.ctypes.data_as(C.POINTER(C.c_int))))
        return [bc[bs[b]:bs[b + 1]].tolist() for b in range(nb)]

    def neighborhood(self, fields=None):
        """ReferenceNeighborhood arrays; `fields` (names) limits which are copied out."""
        want = set(fields) if fields is not None else {"offsets", "neighbor", "r0_len", "e0", "dwdr0", "pair_factor"}
        S = int(lib().orc_slot_count(self._h))
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

        _check(lib().orc_get_neighborhood(self._h, off.ctypes.data_as(C.POINTER(C.c_longlong)), ptr(nb, "neighbor", C.c_int),
                        ptr(ln, "r0_len"), ptr(e0, "e0"), ptr(dw, "dwdr0"), ptr(pf, "pair_factor")))
        out = {"offsets": off, "neighbor": nb, "r0_len": ln, "e0": e0, "dwdr0": dw, "pair_factor": pf}
        return {k: v for k, v in out.items() if k in want or k == "offsets"}

    def set_neighborhood(self, offsets, neighbor, r0_len, e0, dwdr0, pf):
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        nb = np.ascontiguousarray(neighbor, dtype=np.int32)
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (r0_len, e0, dwdr0, pf)]
        _check(lib().orc_set_neighborhood(self._h, off.ctypes.data_as(C.POINTER(C.c_longlong)),
                                          nb.ctypes.data_as(C.POINTER(C.c_int)), *[_dp(a) for a in arrs]))

    # ---- operators
    def correction_matrices(self, threads=1):
        _check(lib().orc_correction_matrices(self._h, threads))

    def deformation_rate(self, threads=1):
        _check(lib().orc_deformation_rate(self._h, threads))

    def update_density(self, threads=1):
        _check(lib().orc_update_density(self._h, threads))

    def momentum_rhs(self, threads=1):
        _check(lib().orc_momentum_rhs(self._h, threads))

    def verlet_step(self, dt, threads=1):
        _check(lib().orc_verlet_step(self._h, dt, threads))

    def apply_constraints(self):
        _check(lib().orc_apply_constraints(self._h))

    def prepare(self, threads=1):
        _check(lib().orc_prepare(self._h, threads))

    def stable_dt(self, h=None):
        out = C.c_double()
        _check(lib().orc_stable_dt(self._h, self.h if h is None else h, C.byref(out)))
        return out.value

    def kinetic_energy(self):
        out = C.c_double()
        _check(lib().orc_kinetic_energy(self._h, C.byref(out)))
        return out.value

    def check_finite(self, step):
        _check(lib().orc_check_finite(self._h, step))

    def damping_sweep(self, scheme, eta_tilde, dt, threads=1):
        _check(lib().orc_damping_sweep(self._h, SCHEMES[scheme], eta_tilde, dt, threads))

    def particle_split_update(self, i, eta, dt_half):
        _check(lib().orc_particle_split_update(self._h, i, eta, dt_half))

    def pairwise_split_update(self, i, slot, eta, dt_half):
        _check(lib().orc_pairwise_split_update(self._h, i, slot, eta, dt_half))

    def explicit_damping_accel(self, eta, threads=1):
        out = np.empty((self.n, self.dim))
        _check(lib().orc_explicit_damping_accel(self._h, eta, _dp(out), threads))
        return out

    def last_run(self):
        """(completed steps, t) of the last run, also when it stopped on an error."""
        out = np.zeros(2)
        _check(lib().orc_last_run(self._h, _dp(out)))
        return int(out[0]), float(out[1])

    def set_contact(self, point, normal, stiffness):
        """ExternalAccel's penalty contact plane (forces.hpp:13-24); stiffness <= 0 removes it."""
        pt = np.zeros(3)
        nm = np.zeros(3)
        pt[: self.dim] = point
        nm[: self.dim] = normal
        _check(lib().orc_set_contact(self._h, _dp(pt), _dp(nm), float(stiffness)))

    def run(self, *, eta, alpha, scheme="particle_split", steps, fixed_dt=0.0, end_time=0.0,
            elastic=True, seed=0, threads=1, resume=False, probe=-1, interval=0.0):
        """runner.cpp:341-391. resume=True continues the previous run (same damping stream, t and
        step count; `steps` is then the cumulative cap; the returned counts are cumulative, the
        times are those of this call). probe >= 0: also the probe series of runner.cpp:328,378-395
        (t, u) at the output marks every `interval` -- returned as "probe" (k x (1 + dim))."""
        params = np.array([self.h, eta, alpha, SCHEMES[scheme], steps, fixed_dt, end_time,
                           1.0 if elastic else 0.0, seed, threads, 1.0 if resume else 0.0,
                           float(probe), float(interval)], dtype=np.float64)
        out = np.zeros(8)
        cap = int(end_time / interval) + 8 if probe >= 0 and interval > 0 else (2 if probe >= 0 else 0)
        samples = np.zeros((max(cap, 1), 4))
        ns = C.c_longlong(0)
        _check(lib().orc_run_probed(self._h, _dp(params), _dp(out), _dp(samples), cap, C.byref(ns)))
        r = {"steps": int(out[0]), "damped": int(out[1]), "t": out[2], "elastic_s": out[3],
             "damping_s": out[4], "total_s": out[5], "last_dt": out[6]}
        if probe >= 0:
            r["probe"] = samples[: ns.value, : 1 + self.dim].copy()
        return r


# ---- the built-in cases (reference: proj/src/tlsph/cases.cpp:15-231)
GRAVITY_CASES = 9.8  # cases.cpp:15 (kGravity)
CLAMP_LAYERS = 3     # cases.cpp:18


def case_spec(name, resolution=0):
    """builtin_cases + make_case (cases.cpp:72-144): the case constants, dp from the resolution."""
    if name in ("bending_cantilever", "twisting_cantilever"):
        spec = dict(name=name, dim=3, resolution=6, length=0.04, thickness=0.016, E=5.0e4, nu=0.45, rho0=1265.0,
                    model="neo_hookean", gravity=GRAVITY_CASES, L=0.04, beta=0.4, end_time=2.0, interval=0.005,
                    probe_target=(0.04, 0.0, 0.0), rotational=False)
        if name == "twisting_cantilever":  # cases.cpp:96-105
            spec.update(resolution=12, gravity=0.0, rotational=True, probe_target=(0.04, 0.008, 0.008))
    elif name == "falling_ball":  # cases.cpp:107-127
        spec = dict(name=name, dim=2, resolution=50, diameter=1.0, clearance=0.25, E=5.0e5, nu=0.45, rho0=1000.0,
                    model="linear_kirchhoff", gravity=GRAVITY_CASES, L=1.0, beta=1.0, end_time=6.0, interval=0.005,
                    probe_target=(0.0, 0.75, 0.0), contact_stiffness=0.0)
    else:
        raise OracleError(2, f"unknown case '{name}'")
    if resolution > 0:
        spec["resolution"] = resolution
    ref = spec["diameter"] if name == "falling_ball" else spec["thickness"]
    spec["dp"] = ref / spec["resolution"]  # cases.cpp:137-141
    return spec


def disk(center, diameter, dp):
    """generate_disk (cases.cpp:48-64): lattice offsets (i dp, j dp), |offset| <= radius, j outer."""
    radius = 0.5 * diameter
    n = int(np.floor(radius / dp))
    pts = []
    for j in range(-n, n + 1):
        for i in range(-n, n + 1):
            ox, oy = i * dp, j * dp
            if np.sqrt(ox * ox + oy * oy) <= radius:
                pts.append((center[0] + ox, center[1] + oy))
    return np.array(pts, dtype=np.float64)


def nearest_particle(r0, target):
    """cases.cpp:146-158: the first particle at the smallest |r0 - target|."""
    d = r0 - np.asarray(target[: r0.shape[1]])
    dist = np.sqrt(np.sum(d * d, axis=1)) if r0.shape[1] == 2 else np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])
    return int(np.argmin(dist))


def case_setup(name, resolution=0):
    """build_case (cases.cpp:160-231) plus the damping the runner derives from the config
    (runner.cpp:146-168: eta from beta = artificial_viscosity, alpha 0.2, seed 0, particle split)."""
    spec = case_spec(name, resolution)
    dp, dim = spec["dp"], spec["dim"]
    mat = material(spec["E"], spec["nu"], spec["rho0"], spec["model"])
    if dim == 3:
        half = 0.5 * spec["thickness"]
        r0 = box_lattice([-CLAMP_LAYERS * dp, -half, -half], [spec["length"], half, half], dp)
        cons = (r0[:, 0] < 0.0).astype(np.uint8)
        body = np.tile([0.0, -spec["gravity"], 0.0], (len(r0), 1))
        if spec["rotational"]:  # rotational_body_force, cases.cpp:66-70,180-186
            # libm sin per particle (math.sin), as std::sin in the reference
            gamma = np.array([(20.0 * GRAVITY_CASES / spec["thickness"]) * math.sin(math.pi * x / (2.0 * spec["length"]))
                              for x in r0[:, 0]])
            body = np.stack([np.zeros(len(r0)), r0[:, 1] * gamma, r0[:, 2] * gamma], axis=1)
            body[cons == 1] = 0.0
        contact = None
    else:
        center = (0.0, spec["clearance"] + 0.5 * spec["diameter"])
        r0 = disk(center, spec["diameter"], dp)
        cons = np.zeros(len(r0), dtype=np.uint8)
        body = np.tile([0.0, -spec["gravity"]], (len(r0), 1))
        k = spec["contact_stiffness"] if spec["contact_stiffness"] > 0 else mat["K"]
        contact = ((0.0, 0.0), (0.0, 1.0), k)
    probe = nearest_particle(r0, spec["probe_target"] if dim == 3 else (0.0, spec["clearance"] + 0.5 * spec["diameter"]))
    eta = artificial_viscosity(spec["beta"], spec["rho0"], spec["E"], spec["L"]) if spec["beta"] > 0 else 0.0
    return dict(spec=spec, r0=r0, V0=dp ** dim, rho0=spec["rho0"], h=1.3 * dp, constrained=cons, body=body,
                material=mat, contact=contact, probe=probe, eta=eta, alpha=0.2, seed=0)


def run_case(name, resolution=0, end_time=None, interval=None, threads=1):
    """The oracle's tlsph_sim_run: case_setup, runner.cpp:299-313 initialisation, the loop of
    :341-391 with the probe series; returns (probe samples, loop result)."""
    c = case_setup(name, resolution)
    spec = c["spec"]
    o = OracleSystem(c["r0"], c["V0"], c["rho0"], c["h"], constrained=c["constrained"])
    o.set_material(spec["E"], spec["nu"], spec["rho0"], spec["model"])
    o.set("body", c["body"])
    if c["contact"] is not None:
        o.set_contact(*c["contact"])
    o.prepare(threads=threads)
    end = spec["end_time"] if end_time is None else end_time
    r = o.run(eta=c["eta"], alpha=c["alpha"], seed=c["seed"], steps=1 << 62, end_time=end, threads=threads,
              probe=c["probe"], interval=spec["interval"] if interval is None else interval)
    return r["probe"], r, o


def probe_csv(samples, dim):
    """write_probe_csv (runner.cpp:422-439): header, then t,u... as %.17g, LF line ends."""
    lines = ["t,ux,uy" if dim == 2 else "t,ux,uy,uz"]
    for row in samples:
        lines.append(",".join("%.17g" % x for x in row[: 1 + dim]))
    return "\n".join(lines) + "\n"


# ---- stateless helpers
def grad_mag(h, dim, r):
    out = C.c_double()
    _check(lib().orc_grad_mag(h, dim, r, C.byref(out)))
    return out.value


def kernel_value(h, dim, r):
    out = C.c_double()
    _check(lib().orc_kernel_value(h, dim, r, C.byref(out)))
    return out.value


def random_uniforms(seed, n):
    out = np.empty(n)
    _check(lib().orc_random_uniforms(seed, n, _dp(out)))
    return out


def random_choice(eta, alpha, seed, n):
    out = np.empty(n)
    _check(lib().orc_random_choice(eta, alpha, seed, n, _dp(out)))
    return out


def viscous_bounds(h, nu_kin, dim):
    out = np.empty(2)
    _check(lib().orc_viscous_bounds(h, nu_kin, dim, _dp(out)))
    return out[0], out[1]


def artificial_viscosity(beta, rho0, E, L):
    out = C.c_double()
    _check(lib().orc_artificial_viscosity(beta, rho0, E, L, C.byref(out)))
    return out.value


def material(E, nu, rho0, model="neo_hookean"):
    out = np.empty(8)
    _check(lib().orc_material(E, nu, rho0, 1 if model == "neo_hookean" else 0, _dp(out)))
    return dict(zip(["lambda", "mu", "K", "G", "E", "nu", "rho0", "c"], out.tolist()))


def second_pk(F, E, nu, rho0, model="neo_hookean"):
    F = np.ascontiguousarray(F, dtype=np.float64)
    d = F.shape[0]
    out = np.empty((d, d))
    _check(lib().orc_second_pk(d, _dp(F), E, nu, rho0, 1 if model == "neo_hookean" else 0, _dp(out)))
    return out


def box_lattice(lo, hi, dp):
    lo = np.ascontiguousarray(lo, dtype=np.float64)
    hi = np.ascontiguousarray(hi, dtype=np.float64)
    d = len(lo)
    n = int(lib().orc_box_lattice(d, _dp(lo), _dp(hi), dp, None))
    if n < 0:
        raise OracleError(1, lib().orc_last_error().decode())
    out = np.empty((n, d))
    lib().orc_box_lattice(d, _dp(lo), _dp(hi), dp, _dp(out))
    return out
