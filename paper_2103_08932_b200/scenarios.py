"""Synthetic benchmark scenarios of BASELINE.json (conventions frozen in BASELINE.md §3).

All inputs are generated on the host with the reference's arithmetic:
  * lattices follow generate_box_lattice (cases.cpp:21-46): counts
    lround(extent/dp), p_d = lo_d + (idx_d + 0.5) dp, x fastest, V0 = dp^D,
    m = rho0 V0;
  * random numbers come from RandomSource (damping.hpp:41-50, std::mt19937_64
    with u = (x >> 11) 2^-53), consumed particle-major / component-minor;
  * h = 1.3 dp, cutoff = cell = 2h, Wendland C2, neo-Hookean rho0 = 1000,
    E = 2e6, nu = 0.3, eta = 0.2 rho0 c h.
No public dataset is involved; these seeded lattices are the configs.
"""
from __future__ import annotations

import math

import numpy as np

from . import dev

RHO0 = 1000.0
E_MOD = 2.0e6
NU = 0.3
GRAVITY = 9.81


def material():
    return dev.Material.from_young_poisson(E_MOD, NU, RHO0, "neo_hookean")


def box_lattice(lo, hi, dp):
    """generate_box_lattice (cases.cpp:21-46)."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    dim = len(lo)
    counts = []
    for d in range(dim):
        extent = hi[d] - lo[d]
        if not extent >= dp * (1.0 - 1e-12):
            raise ValueError(f"degenerate lattice dimension {d}")
        q = extent / dp
        counts.append(max(1, int(math.floor(q + 0.5)) if q >= 0 else -int(math.floor(-q + 0.5))))
    axes = [lo[d] + (np.arange(counts[d], dtype=np.float64) + 0.5) * dp for d in range(dim)]
    grids = np.meshgrid(*axes[::-1], indexing="ij")  # slowest axis first
    pts = np.stack([g.reshape(-1) for g in grids[::-1]], axis=1)  # x fastest
    return np.ascontiguousarray(pts), counts


def eta_for(h):
    c = material().c
    return 0.2 * RHO0 * c * h


def _uniform(seed, n):
    return dev.random_uniforms(seed, n)


def cfg1(scale=1):
    """2D elastic cantilever plate 1.0 x 0.1, dp 0.0025 (400 x 40), left 4 columns clamped."""
    dp = 0.0025 * scale
    r0, counts = box_lattice([0.0, 0.0], [1.0, 0.1], dp)
    n = len(r0)
    h = 1.3 * dp
    u = _uniform(0, n * 2).reshape(n, 2)
    v0 = -0.01 + 0.02 * u
    cons = (r0[:, 0] < 4 * dp).astype(np.uint8)
    body = np.tile([0.0, -GRAVITY], (n, 1))
    return dict(name="cfg1", dim=2, r0=r0, V0=dp * dp, rho0=RHO0, h=h, constrained=cons, v0=v0, body=body,
                eta=eta_for(h), alpha=0.2, seed=0, steps=2000, elastic=True, fixed_dt=0.0, counts=counts)


def box_muller_normals(seed, count):
    """N(0,1) via Box-Muller on RandomSource(seed): z0 = rho cos(2 pi u2), z1 = rho sin(2 pi u2)."""
    pairs = (count + 1) // 2
    u = _uniform(seed, 2 * pairs).reshape(pairs, 2)
    rho = np.sqrt(-2.0 * np.log(1.0 - u[:, 0]))
    z = np.empty((pairs, 2))
    z[:, 0] = rho * np.cos(2.0 * np.pi * u[:, 1])
    z[:, 1] = rho * np.sin(2.0 * np.pi * u[:, 1])
    return z.reshape(-1)[:count]


def cfg2(side=64):
    """3D damping-only sweep: 64^3 lattice on [0,1]^3, v ~ N(0,1), alpha = 1, fixed dt = 0.6 h / c."""
    dp = 1.0 / side
    r0, counts = box_lattice([0.0, 0.0, 0.0], [1.0, 1.0, 1.0], dp)
    n = len(r0)
    h = 1.3 * dp
    v0 = box_muller_normals(1, n * 3).reshape(n, 3)
    c = material().c
    return dict(name="cfg2", dim=3, r0=r0, V0=dp ** 3, rho0=RHO0, h=h, constrained=None, v0=v0, body=None,
                eta=eta_for(h), alpha=1.0, seed=1, steps=500, elastic=False, fixed_dt=0.6 * h / c, counts=counts)


def cfg3(scale=1):
    """3D cantilever beam 4.0 x 0.4 x 0.4, dp 0.01 (400 x 40 x 40), 5-layer clamp, gravity."""
    dp = 0.01 * scale
    r0, counts = box_lattice([0.0, -0.2, -0.2], [4.0, 0.2, 0.2], dp)
    n = len(r0)
    h = 1.3 * dp
    cons = (r0[:, 0] < 5 * dp).astype(np.uint8)
    body = np.tile([0.0, -GRAVITY, 0.0], (n, 1))
    return dict(name="cfg3", dim=3, r0=r0, V0=dp ** 3, rho0=RHO0, h=h, constrained=cons, v0=np.zeros((n, 3)),
                body=body, eta=eta_for(h), alpha=0.2, seed=0, steps=200000, elastic=True, fixed_dt=0.0,
                ke_stop=True, counts=counts)


def cfg4(dp=0.004, extent=(1.0, 1.0, 0.5)):
    """Jittered irregular block (r0 += (2u-1) 0.4 dp from RandomSource(3)), alpha 0.1, 1000 steps."""
    r0, counts = box_lattice([0.0, 0.0, 0.0], list(extent), dp)
    n = len(r0)
    h = 1.3 * dp
    u = _uniform(3, n * 6)
    r0 = r0 + (2.0 * u[: n * 3].reshape(n, 3) - 1.0) * (0.4 * dp)
    v0 = -0.01 + 0.02 * u[n * 3:].reshape(n, 3)
    cons = (r0[:, 0] < 5 * dp).astype(np.uint8)
    body = np.tile([0.0, -GRAVITY, 0.0], (n, 1))
    return dict(name="cfg4", dim=3, r0=np.ascontiguousarray(r0), V0=dp ** 3, rho0=RHO0, h=h, constrained=cons,
                v0=v0, body=body, eta=eta_for(h), alpha=0.1, seed=0, steps=1000, elastic=True, fixed_dt=0.0,
                counts=counts)


def cfg5_weak(layers=250, dp=0.004):
    """Weak-scaling slab: `layers` x-layers of 250 x 250 at dp 0.004 (15.6M particles per GPU)."""
    r0, counts = box_lattice([0.0, 0.0, 0.0], [layers * dp, 1.0, 1.0], dp)
    n = len(r0)
    h = 1.3 * dp
    cons = (r0[:, 0] < 5 * dp).astype(np.uint8)
    body = np.tile([0.0, -GRAVITY, 0.0], (n, 1))
    return dict(name="cfg5", dim=3, r0=r0, V0=dp ** 3, rho0=RHO0, h=h, constrained=cons, v0=np.zeros((n, 3)),
                body=body, eta=eta_for(h), alpha=0.2, seed=0, steps=500, elastic=True, fixed_dt=0.0, counts=counts)


def build_device(cfg, prepare=True):
    """Device system for a scenario, with velocities / body force set and (optionally) the runner init."""
    sys = dev.DeviceSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"], cfg["constrained"])
    sys.set("v", cfg["v0"])
    if cfg.get("body") is not None:
        sys.set("body", cfg["body"])
    if prepare and cfg["elastic"]:
        sys.prepare(material())
    return sys
