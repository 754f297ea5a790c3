"""Regenerate tests/golden/golden.npz (TEST INFRASTRUCTURE ONLY).

The reference (C++/CMake, needs Eigen3 + oneTBB) cannot be built in this image
(DESIGN.md §2), so these vectors come from the CPU oracle AFTER it has been pinned
to every known answer the reference's own suite holds (tests/test_oracle_pins.py).
They freeze the oracle's outputs on fixed seeded inputs so that
  * a later change to the oracle that moves any output is caught on CPU, and
  * the GPU tests have a target that does not depend on the oracle at run time.

Cases (all inputs are regenerated from the parameters stored beside them):
  sweep_{scheme}_{dim}d : 3 Strang damping sweeps (eta_tilde 160, dt 1e-4) on the
      lattices of test_gpu_parity.test_sweep_ordered_bit_exact
      (damping.cpp:53-182 particle split, :91-106/161-176 pairwise split);
  random_choice        : 64 draws of the random-choice damping switch
      (damping.hpp:41-50, damping.cpp:29-34), eta 160, alpha 0.2, seed 7;
  cfg1_loop            : 100 steps of the BASELINE cfg1 loop (runner.cpp:341-391).

Run from the repo root:  python -m tests.golden.make_golden
"""
from __future__ import annotations

import os

import numpy as np

from oracle import oracle as O
from paper_2103_08932_b200 import scenarios as S
from tests.fixtures import lattice_r0, random_velocities

HERE = os.path.dirname(os.path.abspath(__file__))
PATH = os.path.join(HERE, "golden.npz")

SWEEP_COUNTS = {2: [23, 19], 3: [9, 8, 7]}
SWEEP_DP, SWEEP_H, SWEEP_RHO0 = 0.01, 0.013, 1000.0
SWEEP_ETA, SWEEP_DT, SWEEP_N, SWEEP_SEED = 160.0, 1e-4, 3, 43
CFG1_STEPS = 100


def sweep_case(dim):
    r0 = lattice_r0(SWEEP_COUNTS[dim], SWEEP_DP)
    cons = (r0[:, 0] < 0.02).astype(np.uint8)
    v = random_velocities(len(r0), dim, 1.0, SWEEP_SEED)
    v[cons == 1] = 0.0
    return r0, SWEEP_DP ** dim, cons, v


def oracle_sweep(scheme, dim):
    r0, V0, cons, v = sweep_case(dim)
    o = O.OracleSystem(r0, V0, SWEEP_RHO0, SWEEP_H, constrained=cons)
    o.set("v", v)
    for _ in range(SWEEP_N):
        o.damping_sweep(scheme, SWEEP_ETA, SWEEP_DT)
    return o.get("v")


def oracle_cfg1():
    cfg = S.cfg1()
    o = O.OracleSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"], constrained=cfg["constrained"])
    o.set_material(S.E_MOD, S.NU, S.RHO0)
    o.set("v", cfg["v0"])
    o.set("body", cfg["body"])
    o.prepare()
    res = o.run(eta=cfg["eta"], alpha=cfg["alpha"], steps=CFG1_STEPS, seed=cfg["seed"],
                threads=O.openmp_threads())
    return res, o.get("r"), o.get("v")


def generate():
    out = {}
    for dim in (2, 3):
        for scheme in ("particle_split", "pairwise_split"):
            out[f"sweep_{scheme}_{dim}d"] = oracle_sweep(scheme, dim)
    out["random_choice"] = np.asarray(O.random_choice(160.0, 0.2, 7, 64), dtype=np.float64)
    res, r, v = oracle_cfg1()
    out["cfg1_r"], out["cfg1_v"] = r, v
    out["cfg1_scalars"] = np.array([res["steps"], res["damped"], res["t"]], dtype=np.float64)
    return out


if __name__ == "__main__":
    np.savez_compressed(PATH, **generate())
    print("wrote", PATH, os.path.getsize(PATH), "bytes")
