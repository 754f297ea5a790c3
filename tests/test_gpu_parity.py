"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star):
  * cell assignment, cell lists and the neighbour CSR: bit-exact;
  * ORDERED reduction mode: every operator that involves only + - * / sqrt
    (neighbour geometry, B0, dF/dt, damping sweeps, linear-Kirchhoff stress)
    is bit-identical to the oracle;
  * FAST mode and anything downstream of the neo-Hookean log(): relative L2
    error <= 1e-10 (the north_star tolerance for identical sweep order).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2103_08932_b200 import dev
from paper_2103_08932_b200 import scenarios as S
from tests.fixtures import lattice_r0, random_velocities

pytestmark = pytest.mark.gpu

TOL = 1e-10  # north_star: relative L2 for identical sweep order


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


def pair(r0, V0, rho0, h, constrained=None):
    return (O.OracleSystem(r0, V0, rho0, h, constrained=constrained),
            dev.DeviceSystem(r0, V0, rho0, h, constrained=constrained))


def clouds():
    rng = np.random.RandomState(5)
    yield "lattice2d", lattice_r0([23, 17], 0.01), 1e-4, 0.013
    yield "lattice3d", lattice_r0([11, 9, 7], 0.01), 1e-6, 0.013
    yield "random2d", rng.uniform(0, 1, (400, 2)), 1e-4, 0.06
    yield "random3d", rng.uniform(0, 0.5, (500, 3)), 1e-6, 0.05
    base = lattice_r0([10, 10, 10], 0.01)
    yield "jitter3d", base + rng.uniform(-0.004, 0.004, base.shape), 1e-6, 0.013
    r0, _ = S.box_lattice([0.0, 0.0], [1.0, 0.1], 0.0025)  # cfg1 geometry (thin extra cell row)
    yield "cfg1", r0, 0.0025 ** 2, 1.3 * 0.0025


# ---------------------------------------------------------------- splitting cell-linked list
@pytest.mark.parametrize("case", list(clouds()), ids=lambda c: c[0])
def test_cell_grid_and_csr_bit_exact(case):
    _, r0, V0, h = case
    o, d = pair(r0, V0, 1000.0, h)
    go, gd = o.grid(), d.grid()
    assert go["dims"] == gd["dims"]
    assert go["origin"] == gd["origin"]
    assert go["cell_size"] == gd["cell_size"]
    for k in ("cell_of", "cell_start", "cell_particles"):
        assert np.array_equal(go[k], gd[k]), k
    assert o.blocks() == d.blocks()
    no, nd = o.neighborhood(), d.neighborhood()
    for k in ("offsets", "neighbor", "r0_len", "e0", "dwdr0", "pair_factor"):
        assert np.array_equal(no[k], nd[k]), k


def test_block_membership_published_9x6_on_gpu():  # test_neighbors.cpp:95-113
    pts = np.array([[ix + 0.5, iy + 0.5] for iy in range(6) for ix in range(9)])
    d = dev.DeviceSystem(pts, 1.0, 1.0, 0.5)
    assert d.grid()["dims"] == [9, 6]
    blocks = d.blocks()
    assert blocks[0] == [0, 3, 6, 27, 30, 33]
    assert blocks[8] == [20, 23, 26, 47, 50, 53]


def test_interior_count_20_on_gpu():  # test_neighbors.cpp:247-276
    r0 = lattice_r0([12, 12], 0.01)
    d = dev.DeviceSystem(r0, 1e-4, 1.0, 0.013)
    c = int(np.argmin(np.linalg.norm(r0 - [0.06, 0.06], axis=1)))
    off = d.neighborhood()["offsets"]
    assert off[c + 1] - off[c] == 20


def test_coincident_particles_error_text():
    with pytest.raises(dev.TlsphError) as e:
        dev.DeviceSystem(np.array([[0.4, 0.4], [0.1, 0.1], [0.4, 0.4]]), 1.0, 1.0, 0.1)
    assert e.value.kind == "degenerate-geometry"
    assert e.value.message == "coincident particles 0 and 2 in reference configuration"


def test_empty_and_nonfinite_rejected():
    with pytest.raises(dev.TlsphError) as e:
        dev.DeviceSystem(np.zeros((0, 3)), 1.0, 1.0, 0.1)
    assert e.value.kind == "invalid-argument"
    with pytest.raises(dev.TlsphError):
        dev.DeviceSystem(np.array([[0.0, np.nan]]), 1.0, 1.0, 0.1)


# ---------------------------------------------------------------- correction matrices / TL-SPH
@pytest.mark.parametrize("case", list(clouds())[:2] + list(clouds())[4:5], ids=lambda c: c[0])
def test_correction_matrices_bit_exact(case):
    _, r0, V0, h = case
    o, d = pair(r0, V0, 1000.0, h)
    o.correction_matrices()
    d.correction_matrices()
    assert np.array_equal(o.get("B0"), d.get("B0"))


def test_degenerate_b0_error_text():
    d = dev.DeviceSystem(np.array([[0.0, 0.0], [10.0, 0.0]]), 1.0, 1000.0, 0.1)
    with pytest.raises(dev.TlsphError) as e:
        d.correction_matrices()
    assert e.value.message == ("degenerate neighborhood: correction matrix of particle 0 is singular "
                               "or ill-conditioned")


@pytest.mark.parametrize("mode", ["ordered", "fast"])
@pytest.mark.parametrize("dim", [2, 3])
def test_deformation_rate(mode, dim):
    r0 = lattice_r0([9, 8] if dim == 2 else [7, 6, 5], 0.01)
    o, d = pair(r0, 0.01 ** dim, 1000.0, 0.013)
    d.set_reduction(mode)
    o.correction_matrices()
    d.correction_matrices()
    v = random_velocities(len(r0), dim, 1.0, 3)
    o.set("v", v)
    d.set("v", v)
    o.deformation_rate()
    d.deformation_rate()
    if mode == "ordered":
        assert np.array_equal(o.get("dFdt"), d.get("dFdt"))
    else:
        assert rel_l2(d.get("dFdt"), o.get("dFdt")) <= 1e-14


@pytest.mark.parametrize("model", ["linear", "neo_hookean"])
@pytest.mark.parametrize("mode", ["ordered", "fast"])
def test_momentum_rhs(model, mode):
    r0 = lattice_r0([6, 5, 4], 0.01)
    o, d = pair(r0, 1e-6, 1265.0, 0.013)
    d.set_reduction(mode)
    for s in (o, d):
        s.correction_matrices()
    rng = np.random.RandomState(7)
    F = np.eye(3) + rng.uniform(-0.02, 0.02, (len(r0), 3, 3))
    body = np.tile([0.0, -9.8, 0.0], (len(r0), 1))
    for s in (o, d):
        s.set("F", F)
        s.set("body", body)
    o.set_material(5e4, 0.45, 1265.0, model)
    mat = dev.Material.from_young_poisson(5e4, 0.45, 1265.0, model)
    o.momentum_rhs()
    d.momentum_rhs(mat)
    if mode == "ordered" and model == "linear":
        assert np.array_equal(o.get("a"), d.get("a"))
    else:
        assert rel_l2(d.get("a"), o.get("a")) <= 1e-12


def test_update_density_and_inverted_error():
    r0 = lattice_r0([3, 3, 3], 0.01)
    o, d = pair(r0, 1e-6, 1265.0, 0.013)
    F = np.tile(np.eye(3), (27, 1, 1))
    F[0] = np.diag([2.0, 1.0, 1.0])
    for s in (o, d):
        s.set("F", F)
        s.update_density()
    assert np.array_equal(o.get("rho"), d.get("rho"))
    F[2] = -np.eye(3)
    F[5] = -np.eye(3)
    d.set("F", F)
    with pytest.raises(dev.TlsphError) as e:
        d.update_density()
    assert e.value.kind == "inverted-element"
    assert e.value.message == "inverted element: det(F) <= 0 for particle 2"


@pytest.mark.parametrize("model", ["linear", "neo_hookean"])
def test_verlet_step(model):
    r0 = lattice_r0([8, 5, 4], 0.01)
    cons = (r0[:, 0] < 0.02).astype(np.uint8)
    o, d = pair(r0, 1e-6, 1000.0, 0.013, constrained=cons)
    d.set_reduction("ordered")
    o.set_material(2e6, 0.3, 1000.0, model)
    mat = dev.Material.from_young_poisson(2e6, 0.3, 1000.0, model)
    v = random_velocities(len(r0), 3, 0.05, 11)
    body = np.tile([0.0, -9.81, 0.0], (len(r0), 1))
    for s in (o, d):
        s.set("v", v)
        s.set("body", body)
    o.prepare()
    d.prepare(mat)
    for _ in range(20):
        o.verlet_step(1e-5)
        d.verlet_step(mat, 1e-5)
    for k in ("r", "v", "F", "dFdt", "rho", "a"):
        if model == "linear":
            assert np.array_equal(o.get(k), d.get(k)), k
        else:
            assert rel_l2(d.get(k), o.get(k)) <= 1e-12, k


def test_stable_dt_and_kinetic_energy():
    r0 = lattice_r0([5, 5, 5], 0.01)
    o, d = pair(r0, 1e-6, 1000.0, 0.013)
    mat = dev.Material.from_young_poisson(2e6, 0.3, 1000.0)
    o.set_material(2e6, 0.3, 1000.0)
    v = random_velocities(len(r0), 3, 1.0, 2)
    a = random_velocities(len(r0), 3, 50.0, 4)
    for s in (o, d):
        s.set("v", v)
        s.set("a", a)
    assert o.stable_dt(0.013) == d.stable_dt(mat, 0.013)
    assert d.kinetic_energy() == pytest.approx(o.kinetic_energy(), rel=1e-13)


def test_check_finite_message():
    r0 = lattice_r0([4, 4], 0.01)
    d = dev.DeviceSystem(r0, 1e-4, 1000.0, 0.013)
    d.check_finite(3)
    v = np.zeros((16, 2))
    v[7, 1] = np.nan
    v[9, 0] = np.inf
    d.set("v", v)
    with pytest.raises(dev.TlsphError) as e:
        d.check_finite(12)
    assert e.value.kind == "numerical-failure"
    assert e.value.message == "NaN detected at step 12, particle 7"


# ---------------------------------------------------------------- damping sweep
def test_corrected_division_is_ieee_on_device():
    # RN(x/d) via y = RN(1/d) + one Markstein correction, used off the chain
    assert dev.selftest_division(1 << 26, 7) == 0


@pytest.mark.parametrize("scheme", ["particle_split", "pairwise_split"])
@pytest.mark.parametrize("dim", [2, 3])
def test_sweep_ordered_bit_exact(scheme, dim):
    r0 = lattice_r0([23, 19] if dim == 2 else [9, 8, 7], 0.01)
    cons = (r0[:, 0] < 0.02).astype(np.uint8)
    o, d = pair(r0, 0.01 ** dim, 1000.0, 0.013, constrained=cons)
    d.set_reduction("ordered")
    v = random_velocities(len(r0), dim, 1.0, 43)
    v[cons == 1] = 0.0
    o.set("v", v)
    d.set("v", v)
    for _ in range(3):
        o.damping_sweep(scheme, 160.0, 1e-4)
        d.damping_sweep(scheme, 160.0, 1e-4)
    assert np.array_equal(o.get("v"), d.get("v"))


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("scheme", ["particle_split", "pairwise_split"])
def test_sweep_fast_within_tolerance(dim, scheme):
    r0 = lattice_r0([31, 29] if dim == 2 else [13, 12, 11], 0.01)
    o, d = pair(r0, 0.01 ** dim, 1000.0, 0.013)
    v = random_velocities(len(r0), dim, 1.0, 9)
    o.set("v", v)
    d.set("v", v)
    for _ in range(5):
        o.damping_sweep(scheme, 2000.0, 2e-4)
        d.damping_sweep(scheme, 2000.0, 2e-4)
    assert rel_l2(d.get("v"), o.get("v")) <= TOL


def irregular_bodies():
    rng = np.random.RandomState(11)
    yield "random2d", rng.uniform(0, 1, (600, 2)), 1e-4, 0.05          # ragged rows, sparse cells
    yield "random3d", rng.uniform(0, 0.5, (700, 3)), 1e-6, 0.05        # 3D, K <= 4 register path
    base = lattice_r0([12, 10, 9], 0.01)
    yield "jitter3d", base + rng.uniform(-0.004, 0.004, base.shape), 1e-6, 0.013
    yield "dense3d", rng.uniform(0, 0.25, (1000, 3)), 1e-6, 0.05       # > 128 slots per row: generic loop


@pytest.mark.parametrize("case", list(irregular_bodies()), ids=lambda c: c[0])
@pytest.mark.parametrize("mode", ["ordered", "fast"])
@pytest.mark.parametrize("scheme", ["particle_split", "pairwise_split"])
def test_sweep_irregular_bodies(case, mode, scheme):
    """Variable neighbour counts and cell occupancy, including rows longer than the register path."""
    name, r0, V0, h = case
    cons = (r0[:, 0] < np.quantile(r0[:, 0], 0.05)).astype(np.uint8)
    o, d = pair(r0, V0, 1000.0, h, constrained=cons)
    d.set_reduction(mode)
    v = random_velocities(len(r0), r0.shape[1], 1.0, 21)
    v[cons == 1] = 0.0
    o.set("v", v)
    d.set("v", v)
    for _ in range(2):
        o.damping_sweep(scheme, 300.0, 1e-4)
        d.damping_sweep(scheme, 300.0, 1e-4)
    if mode == "ordered":
        assert np.array_equal(o.get("v"), d.get("v"))
    else:
        assert rel_l2(d.get("v"), o.get("v")) <= TOL
    assert np.all(d.get("v")[cons == 1] == 0.0)


@pytest.mark.parametrize("tiling", ["staged", "streamed"])
def test_fast_sweep_follows_clamp_and_mass_changes(tiling):
    """The FAST chain reads its own regrouped copy of the slot rows (bank-spread rows, state.cu
    k_spread_rows: stencil index + clamp bit, pair factor) when every mass is equal, and the
    per-slot / per-stencil mass factors otherwise; the copy must follow clamp flags and masses set
    after construction (damping.cpp:84-86, :151 read them at every sweep)."""
    rng = np.random.RandomState(4)
    base = lattice_r0([14, 12, 10], 0.01)
    r0 = base + rng.uniform(-0.003, 0.003, base.shape)
    n = len(r0)
    o, d = pair(r0, 1e-6, 1000.0, 0.013)
    d.set_reduction("fast")
    d.set_sweep_tiling(tiling)
    v = random_velocities(n, 3, 1.0, 33)

    def sweep_and_compare(cons):
        vv = v.copy()
        vv[cons == 1] = 0.0
        for s in (o, d):
            s.set("v", vv)
        for _ in range(2):
            o.damping_sweep("particle_split", 300.0, 1e-4)
            d.damping_sweep("particle_split", 300.0, 1e-4)
        assert rel_l2(d.get("v"), o.get("v")) <= TOL
        assert np.all(d.get("v")[cons == 1] == 0.0)

    none = np.zeros(n, np.uint8)
    sweep_and_compare(none)                                  # uniform masses, nothing clamped
    cons = (r0[:, 0] < 0.03).astype(np.uint8)
    for s in (o, d):
        s.set("constrained", cons.astype(np.float64))
    sweep_and_compare(cons)                                  # clamp bits rebuilt
    m = 1e-3 * (1.0 + 0.5 * rng.uniform(size=n))
    for s in (o, d):
        s.set("m", m)
    sweep_and_compare(cons)                                  # per-particle masses: slot-order rows
    cons2 = (r0[:, 1] > 0.08).astype(np.uint8)
    for s in (o, d):
        s.set("m", np.full(n, 1e-3))
        s.set("constrained", cons2.astype(np.float64))
    sweep_and_compare(cons2)                                 # uniform again, other clamp set


def test_sweep_zero_eta_noop_and_explicit_rejected():
    r0 = lattice_r0([5, 5], 0.01)
    d = dev.DeviceSystem(r0, 1e-4, 1000.0, 0.013)
    v = random_velocities(25, 2, 1.0, 37)
    d.set("v", v)
    d.damping_sweep("particle_split", 0.0, 1e-4)
    assert np.array_equal(d.get("v"), v)
    with pytest.raises(dev.TlsphError):
        d.damping_sweep("explicit", 1.0, 1e-4)


@pytest.mark.parametrize("scheme", ["particle_split", "pairwise_split"])
def test_sweep_scripted_chain_order(scheme):  # test_damping.cpp:348-436 through the GPU
    dp = 0.01
    r0 = np.array([[(i + 0.5) * dp, 0.5 * dp] for i in range(5)])
    o, d = pair(r0, dp * dp, 1000.0, 1.3 * dp)
    d.set_reduction("ordered")
    v = np.random.RandomState(41).uniform(-1, 1, (5, 2))
    o.set("v", v)
    d.set("v", v)
    o.damping_sweep(scheme, 100.0, 2e-4)
    d.damping_sweep(scheme, 100.0, 2e-4)
    assert np.array_equal(o.get("v"), d.get("v"))


def test_pair_rig_known_answers_on_gpu():  # test_damping.cpp:147-170 with the hand CSR
    r0 = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    csr = {"offsets": [0, 1, 2], "neighbor": [1, 0], "r0_len": [1.0, 1.0],
           "e0": [[1.0, 0, 0], [-1.0, 0, 0]], "dwdr0": [-0.05, -0.05], "pair_factor": [-0.1, -0.1]}
    d = dev.DeviceSystem(r0, 1.0, [1.0, 1.0], 1.0, csr=csr)
    d.set("v", [[1.0, 0.0, 0.0], [0.0, 0.0, 0.0]])
    d.particle_split_update(0, 1.0, 1.0)
    B = -0.1
    diag = B - 1.0
    k = (-B) / (diag * diag + B * B)
    vin = 1.0 + diag * k
    vjn = 0.0 - B * (vin - (0.0 - B * k)) / 1.0
    v = d.get("v")
    assert v[0, 0] == vin and v[1, 0] == vjn
    assert abs(v[0, 0] + v[1, 0] - 1.0) <= 1e-14
    # pairwise 2x2 against the generic solve (test_damping.cpp:219-268)
    rng = np.random.RandomState(19)
    for _ in range(20):
        mi, mj = rng.uniform(0.1, 10.0, 2)
        Bp = rng.uniform(-5.0, -1e-4)
        csr["pair_factor"] = [Bp, Bp]
        d = dev.DeviceSystem(r0, 1.0, [mi, mj], 1.0, csr=csr)
        o = O.OracleSystem(r0, 1.0, [mi, mj], 1.0, build=False)
        o.set_neighborhood(csr["offsets"], csr["neighbor"], csr["r0_len"], csr["e0"], csr["dwdr0"], [Bp, Bp])
        vv = rng.uniform(-2, 2, (2, 3))
        d.set("v", vv)
        o.set("v", vv)
        d.pairwise_split_update(0, 0, 1.0, 1.0)
        o.pairwise_split_update(0, 0, 1.0, 1.0)
        assert np.array_equal(d.get("v"), o.get("v"))


def test_explicit_damping_accel():
    r0 = lattice_r0([7, 6], 0.01)
    o, d = pair(r0, 1e-4, 1000.0, 0.013)
    v = random_velocities(len(r0), 2, 1.0, 13)
    o.set("v", v)
    d.set("v", v)
    assert np.array_equal(o.explicit_damping_accel(20.0), d.explicit_damping_accel(20.0))


def test_sweep_momentum_and_constrained_zero():
    r0 = lattice_r0([12, 11, 10], 0.01)
    cons = (r0[:, 0] < 0.02).astype(np.uint8)
    d = dev.DeviceSystem(r0, 1e-6, 1000.0, 0.013, constrained=cons)
    v = random_velocities(len(r0), 3, 1.0, 47)
    v[cons == 1] = 0.0
    d.set("v", v)
    m = d.get("m")
    free = cons == 0
    p0 = (m[free, None] * v[free]).sum(0)
    d.damping_sweep("particle_split", 160.0, 1e-4)
    out = d.get("v")
    assert np.all(out[cons == 1] == 0.0)
    # momentum of free particles changes only through clamped neighbours' dropped writes
    d2 = dev.DeviceSystem(r0, 1e-6, 1000.0, 0.013)
    v2 = random_velocities(len(r0), 3, 1.0, 48)
    d2.set("v", v2)
    p0 = (m[:, None] * v2).sum(0)
    d2.damping_sweep("particle_split", 160.0, 1e-4)
    p1 = (m[:, None] * d2.get("v")).sum(0)
    assert np.linalg.norm(p1 - p0) <= 1e-10 * (m * np.linalg.norm(v2, axis=1)).sum()


# ---------------------------------------------------------------- BASELINE configs
def test_cfg2_full_size_sweeps_match_oracle():
    cfg = S.cfg2()
    o = O.OracleSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"])
    d = S.build_device(cfg, prepare=False)
    o.set("v", cfg["v0"])
    assert o.neighborhood()["offsets"][-1] == d.slot_count == 20026056
    eta_t = cfg["eta"] / cfg["alpha"]
    for _ in range(2):
        o.damping_sweep("particle_split", eta_t, cfg["fixed_dt"], threads=O.openmp_threads())
        d.damping_sweep("particle_split", eta_t, cfg["fixed_dt"])
    assert rel_l2(d.get("v"), o.get("v")) <= TOL
    # property at full length: variance decays monotonically over 50 more sweeps
    var = [float(d.get("v").var())]
    for _ in range(5):
        d.damping_sweep("particle_split", eta_t, cfg["fixed_dt"], count=10)
        var.append(float(d.get("v").var()))
    assert all(b < a for a, b in zip(var, var[1:]))


def test_cfg1_loop_matches_oracle():
    cfg = S.cfg1()
    mat = S.material()
    o = O.OracleSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"], constrained=cfg["constrained"])
    o.set_material(S.E_MOD, S.NU, S.RHO0)
    o.set("v", cfg["v0"])
    o.set("body", cfg["body"])
    o.prepare()
    d = S.build_device(cfg)
    steps = 200
    ro = o.run(eta=cfg["eta"], alpha=cfg["alpha"], steps=steps, seed=cfg["seed"], threads=O.openmp_threads())
    rd = d.run(mat, eta=cfg["eta"], alpha=cfg["alpha"], steps=steps, seed=cfg["seed"])
    assert rd["steps"] == ro["steps"] == steps
    assert rd["damped"] == ro["damped"]
    assert rd["t"] == pytest.approx(ro["t"], rel=1e-12)
    for k in ("r", "v"):
        assert rel_l2(d.get(k) - (cfg["r0"] if k == "r" else 0), o.get(k) - (cfg["r0"] if k == "r" else 0)) <= TOL, k


def test_loop_end_time_and_nan_failure():
    r0 = lattice_r0([10, 4], 0.01)
    cons = (r0[:, 0] < 0.02).astype(np.uint8)
    mat = dev.Material.from_young_poisson(1e5, 0.3, 1000.0, "linear")
    o = O.OracleSystem(r0, 1e-4, 1000.0, 0.013, constrained=cons)
    o.set_material(1e5, 0.3, 1000.0, "linear")
    d = dev.DeviceSystem(r0, 1e-4, 1000.0, 0.013, constrained=cons)
    body = np.tile([0.0, -9.8], (len(r0), 1))
    o.set("body", body)
    d.set("body", body)
    o.prepare()
    d.prepare(mat)
    ro = o.run(eta=20.0, alpha=0.5, steps=10 ** 9, end_time=0.01, seed=4)
    rd = d.run(mat, eta=20.0, alpha=0.5, end_time=0.01, seed=4)
    assert rd["steps"] == ro["steps"] and rd["damped"] == ro["damped"]
    assert rd["t"] == ro["t"] == pytest.approx(0.01)
    assert rel_l2(d.get("r") - r0, o.get("r") - r0) <= TOL
    # a NaN injected into the state surfaces with the reference message
    v = d.get("v")
    v[17, 0] = np.nan
    d.set("v", v)
    with pytest.raises(dev.TlsphError) as e:
        d.run(mat, eta=20.0, alpha=0.5, steps=5, seed=4)
    assert e.value.kind in ("numerical-failure", "inverted-element")


def tiling_bodies():
    rng = np.random.RandomState(17)
    base3 = lattice_r0([13, 12, 11], 0.01)
    yield "lattice3d_uniform", base3, 0.01 ** 3, 1000.0, 0.013
    yield "lattice3d_masses", base3, 0.01 ** 3, rng.uniform(800.0, 1200.0, len(base3)), 0.013
    base2 = lattice_r0([31, 29], 0.01)
    yield "lattice2d_uniform", base2, 0.01 ** 2, 1000.0, 0.013
    jit = base3 + rng.uniform(-0.004, 0.004, base3.shape)
    yield "jitter3d_masses", jit, rng.uniform(0.5e-6, 1.5e-6, len(jit)), 1000.0, 0.013
    # sparse clouds: ragged rows, empty and single-particle cells, isolated particles
    yield "random2d", rng.uniform(0, 1, (600, 2)), 1e-4, 1000.0, 0.05
    yield "random3d", rng.uniform(0, 0.5, (700, 3)), 1e-6, 1000.0, 0.05


@pytest.mark.parametrize("case", list(tiling_bodies()), ids=lambda c: c[0])
@pytest.mark.parametrize("mode", ["fast", "ordered"])
def test_sweep_tiling_staged_equals_streamed(case, mode):
    """The particle-split sweep's staged (shared-memory slot block) and streamed (L2, register
    prefetch) forms: bitwise-identical results, uniform masses (per-slot clamp bit) and per-particle
    masses (stencil 1/m), with clamped particles. FAST: both within the 1e-10 class of the oracle;
    ORDERED: both equal to the oracle bit for bit."""
    name, r0, V0, rho0, h = case
    cons = (r0[:, 0] < np.quantile(r0[:, 0], 0.1)).astype(np.uint8)
    o = O.OracleSystem(r0, V0, rho0, h, constrained=cons)
    v = random_velocities(len(r0), r0.shape[1], 1.0, 23)
    v[cons == 1] = 0.0
    o.set("v", v)
    for _ in range(3):
        o.damping_sweep("particle_split", 500.0, 1e-4)
    out = {}
    for tiling in ("staged", "streamed"):
        d = dev.DeviceSystem(r0, V0, rho0, h, constrained=cons)
        d.set_reduction(mode)
        d.set_sweep_tiling(tiling)
        d.set("v", v)
        for _ in range(3):
            d.damping_sweep("particle_split", 500.0, 1e-4)
        out[tiling] = d.get("v")
        if mode == "ordered":
            assert np.array_equal(out[tiling], o.get("v")), tiling
        else:
            assert rel_l2(out[tiling], o.get("v")) <= TOL, tiling
        assert np.all(out[tiling][cons == 1] == 0.0)
    assert np.array_equal(out["staged"], out["streamed"])


def test_dense_rows_of_the_streamed_chain_in_a_subprocess():
    """The opt-in dense rows of the streamed FAST chain (TLSPH_SWEEP_DENSE=1: every bank-spread row
    padded to 32 K slots, state.cu k_dense_rows) give the staged form's results bit for bit. The knob is
    read once per process, so the staged-vs-streamed cases above run again in a child with it set."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, TLSPH_SWEEP_DENSE="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(root, "tests", "test_gpu_parity.py"), "-m", "gpu",
                        "-q", "-x", "-k", "staged_equals_streamed and fast"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


def blocking_bodies():
    rng = np.random.RandomState(11)
    base3 = lattice_r0([100, 8, 7], 0.01)
    yield "jitter3d", base3 + rng.uniform(-0.004, 0.004, base3.shape), 0.01 ** 3, 1000.0, 0.013
    base2 = lattice_r0([160, 12], 0.01)
    yield "lattice2d", base2, 0.01 ** 2, 1000.0, 0.013


@pytest.mark.parametrize("case", list(blocking_bodies()), ids=lambda c: c[0])
@pytest.mark.parametrize("mode", ["fast", "ordered"])
@pytest.mark.parametrize("scheme", ["particle_split", "pairwise_split"])
def test_temporally_blocked_sweep_is_bitwise_phase_by_phase(case, mode, scheme):
    """The x-chunked trapezoid schedule of the colour phases (tlsph_dev_set_sweep_blocking) gives the
    phase-by-phase result bit for bit: several chunk widths and depths (uneven chunks, blocks that
    straddle the forward/reverse pass boundary), both tilings, clamped particles; and in the device
    loop (graph-captured sweeps with the device dt)."""
    name, r0, V0, rho0, h = case
    cons = (r0[:, 0] < np.quantile(r0[:, 0], 0.05)).astype(np.uint8)
    v = random_velocities(len(r0), r0.shape[1], 1.0, 29)
    v[cons == 1] = 0.0
    ref = None
    for blocking in ((0, 0), (8, 2), (13, 3), (24, 5)):
        for tiling in (("staged", "streamed") if mode == "fast" and scheme == "particle_split" else ("auto",)):
            d = dev.DeviceSystem(r0, V0, rho0, h, constrained=cons)
            d.set_reduction(mode)
            d.set_sweep_tiling(tiling)
            d.set_sweep_blocking(*blocking)
            d.set("v", v)
            d.damping_sweep(scheme, 400.0, 1e-4, count=2)
            got = d.get("v")
            if ref is None:
                ref = got
                assert d.grid()["dims"][0] >= 30, "body too short to exercise several chunks"
            assert np.array_equal(got, ref), (blocking, tiling)
    if r0.shape[1] == 3 and scheme == "particle_split":
        mat = S.material()
        g = np.zeros_like(r0)
        g[:, 1] = -9.81
        loop = []
        for blocking in ((0, 0), (10, 2)):
            d = dev.DeviceSystem(r0, V0, rho0, h, constrained=cons)
            d.set_reduction(mode)
            d.set_sweep_blocking(*blocking)
            d.set("body", g)
            d.set("v", v * 0.01)
            d.prepare(mat)
            r = d.run(mat, eta=S.eta_for(h), alpha=0.5, steps=6, seed=0)
            loop.append((d.get("v"), d.get("r"), r["damped"]))
        assert loop[0][2] > 0
        assert np.array_equal(loop[0][0], loop[1][0]) and np.array_equal(loop[0][1], loop[1][1])


def test_per_step_resort_is_a_pure_storage_permutation():
    """BASELINE cfg4's per-step re-sort: the device loop rebuilds a current-position cell list every
    step; it matches a host binning of the final positions (bit-exact cells, ascending storage order
    in a cell) and changes no result."""
    dp = 0.01
    base = lattice_r0([10, 8, 6], dp)
    rng = np.random.RandomState(3)
    r0 = base + rng.uniform(-0.4 * dp, 0.4 * dp, base.shape)
    n = len(r0)
    cons = (r0[:, 0] < 2 * dp).astype(np.uint8)
    g = np.zeros_like(r0)
    g[:, 1] = -9.81
    mat = S.material()
    out = {}
    for resort in (False, True):
        d = dev.DeviceSystem(r0, dp ** 3, 1000.0, 1.3 * dp, constrained=cons)
        d.set("body", g)
        d.prepare(mat)
        if resort:
            d.set_resort(True)
        d.run(mat, eta=0.2 * 1000.0 * mat.c * 1.3 * dp, alpha=0.5, steps=25, seed=2)
        out[resort] = (d.get("v"), d.get("r"))
        if resort:
            cs, order = d.current_cells()
            gr = d.grid()
            r = out[True][1]
            origin, cell, dims = np.array(gr["origin"]), gr["cell_size"], np.array(gr["dims"])
            c = np.floor((r - origin) / cell).astype(np.int64)
            c = np.clip(c, 0, dims - 1)
            lin = c[:, 0] + dims[0] * (c[:, 1] + dims[1] * c[:, 2])
            rank = np.empty(n, dtype=np.int64)
            rank[gr["cell_particles"]] = np.arange(n)
            counts = np.bincount(lin, minlength=len(cs) - 1)
            assert np.array_equal(np.diff(cs), counts)
            for k in np.nonzero(counts)[0]:
                ids = np.nonzero(lin == k)[0]
                assert np.array_equal(order[cs[k]:cs[k + 1]], ids[np.argsort(rank[ids])])
    assert np.array_equal(out[False][0], out[True][0]) and np.array_equal(out[False][1], out[True][1])


def test_ke_stop_step_count_matches_reference_path():
    """cfg3's stop rule (KE < ratio x peak KE after the peak) on a reduced-resolution beam (10,000
    particles): FAST and ORDERED stop at the same step (north_star: +-1 %), and the ORDERED state at
    that step matches the oracle run for the same number of steps (relative L2 1e-10)."""
    cfg = S.cfg3(scale=4)
    mat = S.material()
    stops = {}
    for mode in ("ordered", "fast"):
        d = S.build_device(cfg, prepare=True)
        d.set_reduction(mode)
        r = d.run(mat, eta=cfg["eta"], alpha=cfg["alpha"], steps=200000, seed=cfg["seed"], ke_stop=True,
                  ke_ratio=1e-3)
        assert r["stopped_on_ke"]
        stops[mode] = (r["steps"], d.get("v"), d.get("r"))
    n_o, n_f = stops["ordered"][0], stops["fast"][0]
    assert abs(n_f - n_o) <= max(1, 0.01 * n_o)
    o = O.OracleSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"], constrained=cfg["constrained"])
    o.set_material(S.E_MOD, S.NU, S.RHO0)
    o.set("v", cfg["v0"])
    o.set("body", cfg["body"])
    o.prepare(threads=O.openmp_threads())
    ro = o.run(eta=cfg["eta"], alpha=cfg["alpha"], steps=n_o, seed=cfg["seed"], threads=O.openmp_threads())
    assert ro["steps"] == n_o
    assert rel_l2(stops["ordered"][1], o.get("v")) <= TOL
    assert rel_l2(stops["ordered"][2], o.get("r")) <= TOL


@pytest.mark.parametrize("mode", ["fast", "ordered"])
def test_large_body_loop_matches_oracle(mode):
    """Bodies of >= 65,536 particles run the TL-SPH neighbour passes as one thread per particle over
    the group-interleaved slot copy (in both modes): a reduced cfg3 beam (80,000 particles) against
    the oracle, 6 loop steps with random-choice damping."""
    cfg = S.cfg3(scale=2)
    assert len(cfg["r0"]) >= 65536
    mat = S.material()
    d = S.build_device(cfg, prepare=True)
    d.set_reduction(mode)
    r = d.run(mat, eta=cfg["eta"], alpha=0.5, steps=6, seed=cfg["seed"])
    o = O.OracleSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"], constrained=cfg["constrained"])
    o.set_material(S.E_MOD, S.NU, S.RHO0)
    o.set("v", cfg["v0"])
    o.set("body", cfg["body"])
    o.prepare(threads=O.openmp_threads())
    ro = o.run(eta=cfg["eta"], alpha=0.5, steps=6, seed=cfg["seed"], threads=O.openmp_threads())
    assert r["steps"] == ro["steps"] == 6 and r["damped"] == ro["damped"] > 0
    for name in ("v", "r"):
        assert rel_l2(d.get(name), o.get(name)) <= TOL, name


@pytest.mark.parametrize("mode", ["fast", "ordered"])
@pytest.mark.parametrize("tiling", ["staged", "streamed"])
def test_uniform_field_is_exactly_invariant_under_a_stiff_sweep(mode, tiling):
    """tests/test_damping.cpp:336-346 (uniform-field invariance), at the falling-ball's eta~ dt where
    the split sweep amplifies any non-uniformity by ~1e20 per sweep: both modes must leave a uniform
    field bit-for-bit unchanged (FAST forms v_j + bm (v_j - v_i), not (1 + bm) v_j - bm v_i)."""
    c = O.case_setup("falling_ball")
    n = len(c["r0"])
    v = np.tile([0.0, -0.0037], (n, 1))
    d = dev.DeviceSystem(c["r0"], c["V0"], c["rho0"], c["h"], constrained=np.zeros(n, np.uint8))
    d.set_reduction(mode)
    d.set_sweep_tiling(tiling)
    d.set("v", v)
    d.damping_sweep("particle_split", 27950.0, 3.8e-4, count=3)
    assert np.array_equal(d.get("v"), v)
