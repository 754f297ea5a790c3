"""GPU parity at BASELINE size (BASELINE.json configs, conventions of BASELINE.md §3).

The sm_100a path through the C ABI against the CPU oracle (the reference's arithmetic, OpenMP
on the host cores) on the full-size configs:

  * cfg1 (2D plate, 16,000 particles): all 2,000 loop steps, FAST and ORDERED;
  * cfg3 (3D beam, 640,000 particles): the first 20 loop steps, FAST and ORDERED, plus the
    full-size neighbour CSR bit for bit;
  * cfg4 (jittered block, 7.8 M particles): neighbour CSR bit for bit at full size, then the
    first 20 loop steps with the per-step current-cell re-sort on (FAST, the bench's mode);
  * cfg5 weak-scaling share (250 x 250 x 250, 15.6 M particles): two x-slabs with the fused
    peer-store exchange (device-side phase barrier) against the undivided body, bit for bit;
  * a >= 65,536-particle linear-Kirchhoff body (no log(): every operation is + - * / sqrt): the
    slot-order one-thread TL-SPH passes bitwise against the oracle in ORDERED mode, and FAST ==
    ORDERED bitwise (both modes run the same kernels on large bodies).

Bars (north_star): neighbour lists and cells bit-exact; relaxed fields within 1e-10 relative L2
(fp64) for identical sweep order; step and damped-step counts equal.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2103_08932_b200 import dev
from paper_2103_08932_b200 import scenarios as S
from paper_2103_08932_b200 import slabs
from tests.fixtures import assert_slab_field

pytestmark = pytest.mark.gpu

TOL = 1e-10  # north_star: relative L2 for identical sweep order


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


def oracle_for(cfg, material=True):
    o = O.OracleSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"], constrained=cfg["constrained"])
    if material:
        o.set_material(S.E_MOD, S.NU, S.RHO0)
    o.set("v", cfg["v0"])
    if cfg.get("body") is not None:
        o.set("body", cfg["body"])
    return o


def compare_loop(d, o, rd, ro, cfg, steps):
    assert rd["steps"] == ro["steps"] == steps
    assert rd["damped"] == ro["damped"]
    assert rd["t"] == pytest.approx(ro["t"], rel=1e-12)
    assert rel_l2(d.get("v"), o.get("v")) <= TOL, "v"
    assert rel_l2(d.get("r") - cfg["r0"], o.get("r") - cfg["r0"]) <= TOL, "displacement"


@pytest.fixture(scope="module")
def cfg1_oracle():
    cfg = S.cfg1()
    o = oracle_for(cfg)
    threads = O.openmp_threads()
    o.prepare(threads=threads)
    ro = o.run(eta=cfg["eta"], alpha=cfg["alpha"], steps=cfg["steps"], seed=cfg["seed"], threads=threads)
    return cfg, o, ro


@pytest.mark.parametrize("mode", ["fast", "ordered"])
def test_cfg1_full_run_matches_oracle(cfg1_oracle, mode):
    """cfg1 in full: 2,000 steps of the TL-SPH loop with random-choice damping (alpha 0.2)."""
    cfg, o, ro = cfg1_oracle
    d = S.build_device(cfg)
    d.set_reduction(mode)
    rd = d.run(S.material(), eta=cfg["eta"], alpha=cfg["alpha"], steps=cfg["steps"], seed=cfg["seed"])
    compare_loop(d, o, rd, ro, cfg, cfg["steps"])


@pytest.fixture(scope="module")
def cfg3_oracle():
    cfg = S.cfg3()
    o = oracle_for(cfg)
    threads = O.openmp_threads()
    o.prepare(threads=threads)
    ro = o.run(eta=cfg["eta"], alpha=cfg["alpha"], steps=20, seed=cfg["seed"], threads=threads)
    return cfg, o, ro


def test_cfg3_full_size_csr_bit_exact(cfg3_oracle):
    cfg, o, _ = cfg3_oracle
    d = S.build_device(cfg, prepare=False)
    nd, no = d.neighborhood(), o.neighborhood()
    assert len(nd["neighbor"]) == 48_611_784
    for k in ("offsets", "neighbor", "r0_len", "e0", "dwdr0", "pair_factor"):
        assert np.array_equal(nd[k], no[k]), k


@pytest.mark.parametrize("mode", ["fast", "ordered"])
def test_cfg3_full_size_first_20_steps(cfg3_oracle, mode):
    """cfg3 at full resolution (640,000 particles, 48.6 M slots), the first 20 loop steps."""
    cfg, o, ro = cfg3_oracle
    d = S.build_device(cfg)
    d.set_reduction(mode)
    rd = d.run(S.material(), eta=cfg["eta"], alpha=cfg["alpha"], steps=20, seed=cfg["seed"])
    compare_loop(d, o, rd, ro, cfg, 20)


def test_cfg4_full_size_csr_and_first_20_steps():
    """cfg4 at full size: 7,812,500 jittered particles (seed 3). The neighbour CSR (offsets,
    neighbour ids, pair factors) bit for bit, then 20 loop steps (alpha 0.1) with the per-step
    current-cell re-sort on, FAST mode, against the oracle's first 20 steps."""
    cfg = S.cfg4()
    assert len(cfg["r0"]) == 7_812_500
    o = oracle_for(cfg)
    d = S.build_device(cfg, prepare=False)
    nd = d.neighborhood(["neighbor", "pair_factor"])
    no = o.neighborhood(["neighbor", "pair_factor"])
    for k in ("offsets", "neighbor", "pair_factor"):
        assert np.array_equal(nd[k], no[k]), k
    rows = np.diff(no["offsets"])
    assert 40 <= rows.mean() <= 90
    del nd, no
    mat = S.material()
    d.prepare(mat)
    d.set_resort(True)
    threads = O.openmp_threads()
    o.prepare(threads=threads)
    steps = 20
    rd = d.run(mat, eta=cfg["eta"], alpha=cfg["alpha"], steps=steps, seed=cfg["seed"])
    ro = o.run(eta=cfg["eta"], alpha=cfg["alpha"], steps=steps, seed=cfg["seed"], threads=threads)
    compare_loop(d, o, rd, ro, cfg, steps)


@pytest.mark.parametrize("mode", ["ordered", "fast"])
def test_cfg5_weak_share_two_slabs_bitwise_undivided(mode):
    """cfg5's weak-scaling share of one GPU (250^3 lattice, dp 0.004, 5-layer clamp): two x-slabs
    of it with the fused peer-store exchange and the device-side phase barrier give, after two
    sweeps, the velocities of the undivided body, owned and halo columns: bit for bit in ORDERED
    mode, within 1e-12 in FAST mode (a slab's bank-spread rows may sum in another order,
    tests/fixtures.py assert_slab_field)."""
    dp, layers = 0.004, 250
    lo, hi = [0.0, 0.0, 0.0], [layers * dp, 1.0, 1.0]
    h = 1.3 * dp
    r0, _ = S.box_lattice(lo, hi, dp)
    n = len(r0)
    cons = (r0[:, 0] < 5 * dp).astype(np.uint8)
    v = -0.01 + 0.02 * dev.random_uniforms(7, n * 3).reshape(n, 3)
    v[cons == 1] = 0.0
    eta_t, dt = S.eta_for(h) / 0.2, 2e-5
    whole = dev.DeviceSystem(r0, dp ** 3, S.RHO0, h, cons)
    whole.set_reduction(mode)
    whole.set("v", v)
    whole.damping_sweep("particle_split", eta_t, dt, count=2)
    ref = whole.get("v")
    del whole
    systems, parts = [], []
    for rank in range(2):
        grid, ranges, part, r0s = slabs.lattice_slab(lo, hi, dp, h, 2, rank)
        assert np.array_equal(r0s, r0[part.ids])
        d = dev.DeviceSystem(r0s, dp ** 3, S.RHO0, h, cons[part.ids], grid=grid[:2])
        d.set_task_range(part.x0, part.x1)
        d.set_reduction(mode)
        d.set("v", v[part.ids])
        systems.append(d)
        parts.append(part)
    slabs.link_peers(systems)
    slabs.sweep_linked(systems, "particle_split", eta_t, dt, count=2)
    for part, d in zip(parts, systems):
        assert_slab_field(d.get("v"), ref[part.ids], mode)


def test_large_body_linear_kirchhoff_bitwise():
    """>= 65,536 particles (the slot-order one-thread TL-SPH kernels, group-interleaved slot copy)
    with linear Kirchhoff stress: ORDERED equals the oracle bit for bit after 4 loop steps with
    damping; without damping (TL-SPH passes only) FAST equals ORDERED bit for bit, since both
    modes run the same neighbour-pass kernels on large bodies (the FAST sweep is reassociated)."""
    cfg = S.cfg3(scale=2)
    assert len(cfg["r0"]) >= 65536
    mat = dev.Material.from_young_poisson(S.E_MOD, S.NU, S.RHO0, "linear")

    def device_run(mode, eta):
        d = S.build_device(cfg, prepare=False)
        d.set_reduction(mode)
        d.prepare(mat)
        r = d.run(mat, eta=eta, alpha=0.5, steps=4, seed=cfg["seed"])
        return r, [d.get(k) for k in ("v", "r", "F", "dFdt", "a")]

    o = O.OracleSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"], constrained=cfg["constrained"])
    o.set_material(S.E_MOD, S.NU, S.RHO0, model="linear")
    o.set("v", cfg["v0"])
    o.set("body", cfg["body"])
    threads = O.openmp_threads()
    o.prepare(threads=threads)
    ro = o.run(eta=cfg["eta"], alpha=0.5, steps=4, seed=cfg["seed"], threads=threads)
    r, fields = device_run("ordered", cfg["eta"])
    assert r["damped"] == ro["damped"] > 0 and r["t"] == ro["t"]
    for name, got in zip(("v", "r", "F", "dFdt", "a"), fields):
        assert np.array_equal(got, o.get(name)), name
    _, fast = device_run("fast", 0.0)
    _, ordered = device_run("ordered", 0.0)
    for name, a, b in zip(("v", "r", "F", "dFdt", "a"), fast, ordered):
        assert np.array_equal(a, b), name
