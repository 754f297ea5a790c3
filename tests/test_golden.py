"""Committed golden vectors (tests/golden/golden.npz, made by tests/golden/make_golden.py).

CPU: the oracle still reproduces every committed vector bit for bit (guards the
pinned oracle against drift), and the C-ABI random-choice draw matches.
GPU: the sm_100a path, through the C ABI, matches the committed vectors directly
(no oracle call at run time): ORDERED sweeps bitwise, FAST sweeps and the cfg1
loop within the north_star relative-L2 tolerance.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2103_08932_b200 import dev
from paper_2103_08932_b200 import scenarios as S
from tests.golden import make_golden as G

TOL = 1e-10  # north_star: relative L2 for identical sweep order

CASES = [(s, d) for d in (2, 3) for s in ("particle_split", "pairwise_split")]


@pytest.fixture(scope="module")
def golden():
    assert os.path.exists(G.PATH), "tests/golden/golden.npz missing: python -m tests.golden.make_golden"
    return dict(np.load(G.PATH))


def rel_l2(a, b):
    a, b = np.ravel(a), np.ravel(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("scheme,dim", CASES)
def test_oracle_reproduces_golden_sweeps(golden, scheme, dim):
    assert np.array_equal(G.oracle_sweep(scheme, dim), golden[f"sweep_{scheme}_{dim}d"])


def test_random_choice_golden(golden):
    assert np.array_equal(O.random_choice(160.0, 0.2, 7, 64), golden["random_choice"])
    assert np.array_equal(dev.random_choice(160.0, 0.2, 7, 64), golden["random_choice"])


def test_oracle_reproduces_golden_cfg1_loop(golden):
    res, r, v = G.oracle_cfg1()
    assert [res["steps"], res["damped"], res["t"]] == list(golden["cfg1_scalars"])
    assert np.array_equal(r, golden["cfg1_r"]) and np.array_equal(v, golden["cfg1_v"])


def _device_sweep(scheme, dim, mode):
    r0, V0, cons, v = G.sweep_case(dim)
    d = dev.DeviceSystem(r0, V0, G.SWEEP_RHO0, G.SWEEP_H, constrained=cons)
    d.set_reduction(mode)
    d.set("v", v)
    for _ in range(G.SWEEP_N):
        d.damping_sweep(scheme, G.SWEEP_ETA, G.SWEEP_DT)
    return d.get("v")


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,dim", CASES)
def test_gpu_ordered_sweep_equals_golden(golden, scheme, dim):
    assert np.array_equal(_device_sweep(scheme, dim, "ordered"), golden[f"sweep_{scheme}_{dim}d"])


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,dim", CASES)
def test_gpu_fast_sweep_within_tolerance_of_golden(golden, scheme, dim):
    assert rel_l2(_device_sweep(scheme, dim, "fast"), golden[f"sweep_{scheme}_{dim}d"]) <= TOL


@pytest.mark.gpu
def test_gpu_cfg1_loop_matches_golden(golden):
    cfg = S.cfg1()
    d = S.build_device(cfg)
    rd = d.run(S.material(), eta=cfg["eta"], alpha=cfg["alpha"], steps=G.CFG1_STEPS, seed=cfg["seed"])
    steps, damped, t = golden["cfg1_scalars"]
    assert rd["steps"] == steps and rd["damped"] == damped
    assert rd["t"] == pytest.approx(t, rel=1e-12)
    assert rel_l2(d.get("r") - cfg["r0"], golden["cfg1_r"] - cfg["r0"]) <= TOL
    assert rel_l2(d.get("v"), golden["cfg1_v"]) <= TOL
