"""Pins the CPU oracle to the reference's own known-answer tests.

The reference cannot be built here (Eigen3/oneTBB absent), so the oracle is
pinned against every known answer and property its test suite holds for the
hot path. Each test names the reference test it ports.
These run on CPU only (no GPU marker).
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from tests.fixtures import (lattice_r0, random_velocities, oracle_deformation_rate, oracle_momentum_accel,
                            oracle_viscous_accel, total_momentum, momentum_scale)


def approx(expected, eps):
    """doctest::Approx(expected).epsilon(eps): |a-b| < eps * (1 + max(|a|, |b|))."""
    class _A:
        def __eq__(self, got):
            return abs(got - expected) < eps * (1.0 + max(abs(got), abs(expected)))

        def __repr__(self):
            return f"Approx({expected!r}, eps={eps})"
    return _A()


def lattice_system(counts, dp, rho0, build=True):
    r0 = lattice_r0(counts, dp)
    dim = len(counts)
    return O.OracleSystem(r0, dp ** dim, rho0, 1.3 * dp, build=build)


def pair_rig(m_i, m_j, pair_factor):
    """test_damping.cpp:18-34: two particles, hand-built CSR."""
    r0 = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    s = O.OracleSystem(r0, 1.0, [m_i, m_j], 1.0, build=False)
    s.set_neighborhood([0, 1, 2], [1, 0], [1.0, 1.0], [[1.0, 0, 0], [-1.0, 0, 0]],
                       [pair_factor / 2.0, pair_factor / 2.0], [pair_factor, pair_factor])
    return s


# ------------------------------------------------------------------ damping (test_damping.cpp)
def test_artificial_viscosity_published_values():  # :38-44
    assert O.artificial_viscosity(0.4, 1265.0, 5.0e4, 0.04) == approx(31.8, 2e-3)
    assert O.artificial_viscosity(1.0, 1000.0, 5.0e5, 1.0) == approx(5590.0, 1e-3)
    assert O.artificial_viscosity(0.0, 1000.0, 5.0e5, 1.0) == 0.0


def test_viscous_bounds():  # :46-63
    for h in (0.2, 1.0):
        for nu in (0.3, 4.0):
            for dim in (1, 2, 3):
                e, i = O.viscous_bounds(h, nu, dim)
                assert i / e == approx(100.0, 1e-14)
    e, i = O.viscous_bounds(1.0, 1.0, 1)
    assert e == approx(0.5, 1e-14) and i == approx(50.0, 1e-14)
    e, _ = O.viscous_bounds(0.00867, 32.0 / 1265.0, 3)
    assert e == approx(4.95e-4, 2e-3)


def test_random_choice_alpha_one():  # :65-70
    assert np.all(O.random_choice(32.0, 1.0, 99, 1000) == 32.0)


def test_random_choice_fraction_and_mean():  # :72-90
    vals = O.random_choice(32.0, 0.2, 42, 100000)
    applied = vals > 0
    assert np.all(np.abs(vals[applied] - 160.0) <= 1e-14 * 160.0)
    assert abs(applied.mean() - 0.2) <= 0.01
    assert abs(vals.mean() - 32.0) <= 0.02 * 32.0


def test_random_source_reproducible_and_bad_alpha():  # :92-100
    assert np.array_equal(O.random_uniforms(7, 100), O.random_uniforms(7, 100))
    for alpha in (0.0, 1.5):
        with pytest.raises(O.OracleError):
            O.random_choice(1.0, alpha, 1, 1)


def test_random_source_mapping_mt19937_64():
    # std::mt19937_64 default-seed 10000th output is fixed by the C++ standard
    # ([rand.predef]: 9981545732273789042); u = (x >> 11) * 2^-53.
    u = O.random_uniforms(5489, 10000)
    assert u[-1] == (9981545732273789042 >> 11) * 2.0 ** -53


def test_explicit_damping_uniform_momentum_oracle():  # :102-129
    s = lattice_system([5, 2], 0.01, 1000.0)
    s.set("v", np.tile([0.7, -0.3], (s.n, 1)))
    assert np.all(np.linalg.norm(s.explicit_damping_accel(20.0), axis=1) == 0.0)
    v = random_velocities(s.n, 2, 1.0, 13)
    s.set("v", v)
    acc = s.explicit_damping_accel(20.0)
    m = s.get("m")
    total = (m[:, None] * acc).sum(0)
    assert np.linalg.norm(total) <= 1e-12 * (m * np.linalg.norm(acc, axis=1)).sum()
    ref = oracle_viscous_accel(s.get("r0"), v, s.get("V0"), m, s.h, 20.0)
    assert np.all(np.linalg.norm(acc - ref, axis=1) <= 1e-12 * (1 + np.linalg.norm(ref, axis=1)))


def test_particle_split_noop_cases():  # :131-145
    rig = pair_rig(1.0, 1.0, -0.1)
    rig.set("v", [[0.3, 0.2, -0.1], [0.3, 0.2, -0.1]])
    rig.particle_split_update(0, 1.0, 1.0)
    assert np.all(rig.get("v") == np.array([[0.3, 0.2, -0.1]] * 2))
    lonely = O.OracleSystem(np.zeros((1, 3)), 1.0, 1.0, 1.0, build=False)
    lonely.set_neighborhood([0, 0], np.zeros(0), np.zeros(0), np.zeros((0, 3)), np.zeros(0), np.zeros(0))
    lonely.set("v", [[1.0, 0.0, 0.0]])
    lonely.particle_split_update(0, 1.0, 1.0)
    assert np.all(lonely.get("v") == [[1.0, 0.0, 0.0]])


def test_particle_split_scalar_rederivation():  # :147-170
    rig = pair_rig(1.0, 1.0, -0.1)
    rig.set("v", [[1.0, 0.0, 0.0], [0.0, 0.0, 0.0]])
    rig.particle_split_update(0, 1.0, 1.0)
    B = -0.1
    diag = B - 1.0
    E = -B * 1.0
    k = E / (diag * diag + B * B)
    vin = 1.0 + diag * k
    vjp = 0.0 - B * k
    vjn = 0.0 - B * (vin - vjp) / 1.0
    v = rig.get("v")
    assert v[0, 0] == approx(vin, 1e-14)
    assert v[1, 0] == approx(vjn, 1e-14)
    assert vin == approx(1.0 - 1.1 * 0.1 / 1.22, 1e-12)
    assert v[0, 0] + v[1, 0] == approx(1.0, 1e-14)


def test_particle_split_momentum_and_implicit_residual():  # :172-217
    s = lattice_system([8, 8], 0.01, 1000.0)
    s.set("v", random_velocities(s.n, 2, 1.0, 17))
    nb = s.neighborhood()
    m = s.get("m")
    eta, dth = 200.0, 1e-3
    rng = np.random.RandomState(17)
    for _ in range(200):
        i = int(rng.randint(0, s.n))
        lo, hi = nb["offsets"][i], nb["offsets"][i + 1]
        if lo == hi:
            continue
        vb = s.get("v")
        p0 = total_momentum(m, vb)
        s.particle_split_update(i, eta, dth)
        va = s.get("v")
        assert np.linalg.norm(total_momentum(m, va) - p0) <= 1e-10 * momentum_scale(m, va)
        b = eta * nb["pair_factor"][lo:hi] * dth
        js = nb["neighbor"][lo:hi]
        residual = -(b[:, None] * (vb[i] - vb[js])).sum(0)
        diag = b.sum() - m[i]
        dvi = va[i] - vb[i]
        k = dvi / diag
        recon = diag * dvi - (b[:, None] * (-b[:, None] * k)).sum(0)
        assert np.linalg.norm(recon - residual) <= 1e-12 * (1 + np.linalg.norm(residual))
        assert np.linalg.norm(k - residual / (diag * diag + (b * b).sum())) <= 1e-12 * (1 + np.linalg.norm(k))


def test_pairwise_solves_2x2_exactly():  # :219-268
    rng = np.random.RandomState(19)
    for _ in range(500):
        mi, mj = rng.uniform(0.1, 10.0, 2)
        B = rng.uniform(-5.0, -1e-4)
        rig = pair_rig(mi, mj, B)
        v = rng.uniform(-2, 2, (2, 3))
        rig.set("v", v)
        rig.pairwise_split_update(0, 0, 1.0, 1.0)
        va = rig.get("v")
        dvi, dvj = va[0] - v[0], va[1] - v[1]
        vij = v[0] - v[1]
        a11, a12, a21, a22 = mi - B, B, B, mj - B
        det = a11 * a22 - a12 * a21
        for d in range(3):
            x = vij[d]
            assert dvi[d] == approx((B * x * a22 - a12 * (-B * x)) / det, 1e-12)
            assert dvj[d] == approx((a11 * (-B * x) - B * x * a21) / det, 1e-12)
        lhs = mi * dvi
        rhs = B * (vij + dvi - dvj)
        assert np.linalg.norm(lhs - rhs) <= 1e-12 * (1 + np.linalg.norm(rhs))
        p0 = mi * v[0] + mj * v[1]
        p1 = mi * va[0] + mj * va[1]
        assert np.linalg.norm(p1 - p0) <= 1e-12 * (1 + np.linalg.norm(p0))


def test_pairwise_shrinks_relative_velocity_and_energy():  # :270-293
    rng = np.random.RandomState(23)
    for _ in range(1000):
        mi, mj = rng.uniform(0.1, 10.0, 2)
        rig = pair_rig(mi, mj, rng.uniform(-5.0, -1e-4))
        v = rng.uniform(-2, 2, (2, 3))
        rig.set("v", v)
        ke0 = rig.kinetic_energy()
        rig.pairwise_split_update(0, 0, 1.0, 1.0)
        va = rig.get("v")
        assert rig.kinetic_energy() <= ke0 * (1 + 1e-14)
        assert np.linalg.norm(va[0] - va[1]) <= np.linalg.norm(v[0] - v[1]) * (1 + 1e-14)


@pytest.mark.parametrize("scheme", ["particle_split", "pairwise_split"])
def test_full_sweep_conserves_momentum(scheme):  # :295-307
    s = lattice_system([9, 9], 0.01, 1000.0)
    s.set("v", random_velocities(s.n, 2, 1.0, 29))
    m = s.get("m")
    p0 = total_momentum(m, s.get("v"))
    scale = momentum_scale(m, s.get("v"))
    s.damping_sweep(scheme, 160.0, 1e-4)
    assert np.linalg.norm(total_momentum(m, s.get("v")) - p0) <= 1e-10 * scale


def test_pairwise_sweeps_never_increase_energy():  # :309-321
    s = lattice_system([6, 6], 0.01, 1000.0)
    rng = np.random.RandomState(31)
    for _ in range(1000):
        s.set("v", rng.uniform(-1, 1, (s.n, 2)))
        e0 = s.kinetic_energy()
        s.damping_sweep("pairwise_split", 300.0, 5e-4)
        assert s.kinetic_energy() <= e0 * (1 + 1e-14)


def test_zero_eta_is_noop():  # :323-334
    s = lattice_system([5, 5], 0.01, 1000.0)
    v = random_velocities(s.n, 2, 1.0, 37)
    s.set("v", v)
    s.damping_sweep("particle_split", 0.0, 1e-4)
    assert np.array_equal(s.get("v"), v)


@pytest.mark.parametrize("scheme", ["particle_split", "pairwise_split"])
def test_uniform_velocity_invariant(scheme):  # :336-346
    s = lattice_system([4, 4, 4], 0.01, 1265.0)
    s.set("v", np.tile([0.2, -0.5, 0.9], (s.n, 1)))
    s.damping_sweep(scheme, 160.0, 1e-4)
    assert np.all(np.linalg.norm(s.get("v") - [0.2, -0.5, 0.9], axis=1) <= 1e-15)


@pytest.mark.parametrize("scheme", ["particle_split", "pairwise_split"])
def test_sweep_order_matches_scripted_chain(scheme):  # :348-436
    dp = 0.01
    r0 = np.array([[(i + 0.5) * dp, 0.5 * dp] for i in range(5)])
    s = O.OracleSystem(r0, dp * dp, 1000.0, 1.3 * dp)
    g = s.grid()
    assert len(g["cell_start"]) - 1 == 2
    assert g["cell_particles"][g["cell_start"][0]:g["cell_start"][1]].tolist() == [0, 1, 2]
    assert g["cell_particles"][g["cell_start"][1]:g["cell_start"][2]].tolist() == [3, 4]
    nb = s.neighborhood()
    rng = np.random.RandomState(41)
    v0 = rng.uniform(-1, 1, (5, 2))
    s.set("v", v0)
    eta, dt = 100.0, 2e-4
    s.damping_sweep(scheme, eta, dt)
    m = s.get("m")
    rv = v0.copy()

    def particle_split(i, tau):
        lo, hi = nb["offsets"][i], nb["offsets"][i + 1]
        if lo == hi:
            return
        res = np.zeros(2)
        sb = sb2 = 0.0
        for sl in range(lo, hi):
            j = nb["neighbor"][sl]
            b = eta * nb["pair_factor"][sl] * tau
            res -= b * (rv[i] - rv[j])
            sb += b
            sb2 += b * b
        diag = sb - m[i]
        k = res / (diag * diag + sb2)
        vin = rv[i] + diag * k
        for sl in range(lo, hi):
            j = nb["neighbor"][sl]
            b = eta * nb["pair_factor"][sl] * tau
            pred = rv[j] - b * k
            rv[j] -= (b / m[j]) * (vin - pred)
        rv[i] = vin

    def pair(i, sl, tau):
        j = nb["neighbor"][sl]
        b = eta * nb["pair_factor"][sl] * tau
        vij = rv[i] - rv[j]
        den = m[i] * m[j] - (m[i] + m[j]) * b
        rv[i] += m[j] * (b / den) * vij
        rv[j] -= m[i] * (b / den) * vij

    for idx in [0, 1, 2, 3, 4, 4, 3, 2, 1, 0]:
        if scheme == "particle_split":
            particle_split(idx, 0.5 * dt)
        else:
            lo, hi = nb["offsets"][idx], nb["offsets"][idx + 1]
            for sl in range(lo, hi):
                pair(idx, sl, 0.25 * dt)
            for sl in range(hi - 1, lo - 1, -1):
                pair(idx, sl, 0.25 * dt)
    out = s.get("v")
    assert np.all(np.linalg.norm(out - rv, axis=1) <= 1e-14 * (1 + np.linalg.norm(rv, axis=1)))


@pytest.mark.parametrize("scheme", ["particle_split", "pairwise_split"])
def test_parallel_sweep_bitwise_equals_serial(scheme):  # :438-456
    if O.openmp_threads() < 2:
        pytest.skip("single hardware thread")
    a = lattice_system([45, 45], 0.01, 1000.0)
    b = lattice_system([45, 45], 0.01, 1000.0)
    v = random_velocities(a.n, 2, 1.0, 43)
    a.set("v", v)
    b.set("v", v)
    a.damping_sweep(scheme, 160.0, 1e-4, threads=1)
    b.damping_sweep(scheme, 160.0, 1e-4, threads=4)
    assert np.array_equal(a.get("v"), b.get("v"))


def test_constrained_stay_zero():  # :458-476
    r0 = lattice_r0([8, 4], 0.01)
    cons = (r0[:, 0] < 0.02).astype(np.uint8)
    s = O.OracleSystem(r0, 1e-4, 1000.0, 0.013, constrained=cons)
    s.set("v", random_velocities(s.n, 2, 1.0, 47))
    s.apply_constraints()
    for scheme in ("particle_split", "pairwise_split"):
        s.damping_sweep(scheme, 160.0, 1e-4)
        assert np.all(np.linalg.norm(s.get("v")[cons == 1], axis=1) == 0.0)


# ------------------------------------------------------------------ neighbours (test_neighbors.cpp)
def test_single_particle_one_cell():  # :43-48
    s = O.OracleSystem(np.array([[0.3, 0.7]]), 1.0, 1.0, 0.25)
    g = s.grid()
    assert len(g["cell_start"]) - 1 == 1 and g["cell_particles"].tolist() == [0]


def test_empty_particle_set_rejected():  # :50-53
    with pytest.raises(O.OracleError):
        O.OracleSystem(np.zeros((0, 2)), 1.0, 1.0, 0.25)


def test_distant_particles_not_neighbours():  # :55-64
    s = O.OracleSystem(np.array([[0.0, 0, 0], [0.25, 0, 0]]), 1.0, 1.0, 0.05)
    nb = s.neighborhood()
    assert nb["offsets"].tolist() == [0, 0, 0]


def test_stencil_candidates_cover_bruteforce():  # :66-93
    rng = np.random.RandomState(5)
    pts = rng.uniform(0, 1, (200, 2))
    s = O.OracleSystem(pts, 1.0, 1.0, 0.06)
    nb = s.neighborhood()
    diff = pts[:, None] - pts[None]
    dist = np.sqrt((diff ** 2).sum(-1))
    np.fill_diagonal(dist, np.inf)
    exact = {(i, j) for i, j in zip(*np.nonzero(dist < 0.12))}
    got = {(i, int(nb["neighbor"][k])) for i in range(200) for k in range(nb["offsets"][i], nb["offsets"][i + 1])}
    assert got == exact


def test_block_membership_published_9x6():  # :95-113
    pts = np.array([[ix + 0.5, iy + 0.5] for iy in range(6) for ix in range(9)])
    s = O.OracleSystem(pts, 1.0, 1.0, 0.5)
    g = s.grid()
    assert g["dims"] == [9, 6]
    blocks = s.blocks()
    assert len(blocks) == 9
    assert blocks[0] == [0, 3, 6, 27, 30, 33]
    assert blocks[8] == [20, 23, 26, 47, 50, 53]


@pytest.mark.parametrize("dim", [2, 3])
def test_blocks_partition_with_residue_colouring(dim):  # :115-154 and :156-196
    rng = np.random.RandomState(23 + dim)
    for _ in range(6):
        hi = rng.randint(1, 13, dim) - 0.01
        s = O.OracleSystem(np.array([np.zeros(dim), hi]), 1.0, 1.0, 0.5)
        g = s.grid()
        dims = g["dims"]
        blocks = s.blocks()
        assert len(blocks) == 3 ** dim
        seen = np.zeros(int(np.prod(dims)), dtype=int)

        def coords(c):
            out = []
            for d in range(dim):
                out.append(c % dims[d])
                c //= dims[d]
            return np.array(out)

        for blk in blocks:
            assert blk == sorted(blk)
            cs = [coords(c) for c in blk]
            for c in blk:
                seen[c] += 1
            for a in range(len(cs)):
                for b in range(a + 1, len(cs)):
                    assert np.all((cs[a] - cs[b]) % 3 == 0)
                    assert np.any(np.abs(cs[a] - cs[b]) > 2)  # stencils disjoint
        assert np.all(seen == 1)


def test_neighbourhoods_symmetric_nonpositive():  # :198-224
    rng = np.random.RandomState(31)
    pts = rng.uniform(0, 0.5, (120, 3))
    s = O.OracleSystem(pts, 1e-6, 1.0, 0.05)
    nb = s.neighborhood()
    off = nb["offsets"]
    for i in range(120):
        row = nb["neighbor"][off[i]:off[i + 1]]
        assert np.all(np.diff(row) > 0)
        for k in range(off[i], off[i + 1]):
            j = nb["neighbor"][k]
            assert nb["pair_factor"][k] <= 0.0
            back = [t for t in range(off[j], off[j + 1]) if nb["neighbor"][t] == i]
            assert len(back) == 1
            assert nb["r0_len"][back[0]] == nb["r0_len"][k]
            assert np.linalg.norm(nb["e0"][back[0]] + nb["e0"][k]) <= 1e-15


def test_isolated_and_close_pair():  # :226-236
    h = 0.1
    s = O.OracleSystem(np.array([[0.0, 0.0], [h, 0.0], [5.0, 5.0]]), 1.0, 1.0, h)
    nb = s.neighborhood()
    assert np.diff(nb["offsets"]).tolist() == [1, 1, 0]
    assert nb["dwdr0"][0] < 0.0


def test_coincident_particles_degenerate():  # :238-245
    with pytest.raises(O.OracleError) as e:
        O.OracleSystem(np.array([[0.4, 0.4], [0.4, 0.4]]), 1.0, 1.0, 0.1)
    assert e.value.kind == "degenerate-geometry"
    assert "coincident particles 0 and 1" in e.value.message


def test_lattice_interior_count_20():  # :247-276
    s = lattice_system([12, 12], 0.01, 1.0)
    r0 = s.get("r0")
    c = int(np.argmin(np.linalg.norm(r0 - [0.06, 0.06], axis=1)))
    nb = s.neighborhood()
    assert nb["offsets"][c + 1] - nb["offsets"][c] == 20


def test_block_sweep_reverse_is_mirror():  # :278-326 (structure of the schedule)
    pts = np.array([[ix + 0.5, iy + 0.5] for iy in range(5) for ix in range(7)])
    s = O.OracleSystem(pts, 1.0, 1.0, 0.5)
    blocks = s.blocks()
    forward = [c for b in blocks for c in b]
    reverse = [c for b in reversed(blocks) for c in reversed(b)]
    assert reverse == forward[::-1]
    assert sorted(forward) == list(range(len(s.grid()["cell_start"]) - 1))


# ------------------------------------------------------------------ integrator (test_integrator.cpp)
def test_linear_completeness():  # :15-30
    s = lattice_system([10, 10], 0.01, 1000.0)
    s.correction_matrices()
    L = np.array([[0.3, -1.2], [0.7, 0.4]])
    s.set("v", s.get("r0") @ L.T)
    s.deformation_rate()
    d = s.get("dFdt")
    assert np.all(np.sqrt(((d - L) ** 2).sum((1, 2))) <= 1e-10 * np.sqrt((L ** 2).sum()))


def test_correction_matrix_matches_direct_inverse():  # :32-67
    s = lattice_system([12, 12], 0.005, 1000.0)
    s.correction_matrices()
    r0 = s.get("r0")
    c = int(np.argmin(np.linalg.norm(r0 - [0.03, 0.03], axis=1)))
    from tests.fixtures import wendland_grad
    mom = np.zeros((2, 2))
    for j in range(s.n):
        if j == c:
            continue
        diff = r0[c] - r0[j]
        dist = np.linalg.norm(diff)
        if dist >= 2 * s.h:
            continue
        grad = wendland_grad(s.h, 2, dist) * diff / dist
        mom -= 0.005 ** 2 * np.outer(diff, grad)
    det = mom[0, 0] * mom[1, 1] - mom[0, 1] * mom[1, 0]
    inv = np.array([[mom[1, 1], -mom[0, 1]], [-mom[1, 0], mom[0, 0]]]) / det
    B0 = s.get("B0")[c]
    assert np.sqrt(((B0 - inv) ** 2).sum()) <= 1e-12
    assert np.sqrt(((B0 - np.eye(2)) ** 2).sum()) < 0.05


def test_particle_without_neighbours_fails():  # :69-80
    s = O.OracleSystem(np.array([[0.0, 0.0], [10.0, 0.0]]), 1.0, 1000.0, 0.1)
    with pytest.raises(O.OracleError) as e:
        s.correction_matrices()
    assert e.value.kind == "degenerate-geometry"
    assert "particle 0" in e.value.message


def test_uniform_velocity_zero_rate():  # :82-90
    s = lattice_system([4, 4, 4], 0.01, 1265.0)
    s.correction_matrices()
    s.set("v", np.tile([0.4, -0.2, 1.0], (s.n, 1)))
    s.deformation_rate()
    assert np.all(s.get("dFdt") == 0.0)


def test_deformation_rate_bruteforce():  # :92-106
    s = lattice_system([7, 7], 0.02, 1000.0)
    s.correction_matrices()
    v = random_velocities(s.n, 2, 1.0, 3)
    s.set("v", v)
    s.deformation_rate()
    ref = oracle_deformation_rate(s.get("r0"), v, s.get("V0"), s.get("B0"), s.h)
    got = s.get("dFdt")
    assert np.all(np.sqrt(((got - ref) ** 2).sum((1, 2))) <= 1e-12 * (1 + np.sqrt((ref ** 2).sum((1, 2)))))


def test_density_follows_det():  # :108-133
    s = lattice_system([3, 3, 3], 0.01, 1265.0)
    s.update_density()
    assert s.get("rho")[0] == approx(1265.0, 1e-14)
    F = s.get("F")
    F[0] = np.diag([2.0, 1.0, 1.0])
    s.set("F", F)
    s.update_density()
    assert s.get("rho")[0] == approx(632.5, 1e-14)
    F[2] = -np.eye(3)
    s.set("F", F)
    with pytest.raises(O.OracleError) as e:
        s.update_density()
    assert e.value.message == "inverted element: det(F) <= 0 for particle 2"


def test_momentum_stress_free_only_body_force():  # :135-151
    s = lattice_system([5, 3, 3], 0.01, 1265.0)
    s.correction_matrices()
    s.set_material(5e4, 0.45, 1265.0, "neo_hookean")
    s.momentum_rhs()
    assert np.all(s.get("a") == 0.0)
    s.set("body", np.tile([0.0, -9.8, 0.0], (s.n, 1)))
    s.momentum_rhs()
    assert np.all(np.linalg.norm(s.get("a") - [0, -9.8, 0], axis=1) <= 1e-12 * 9.8)


def test_internal_forces_conserve_momentum():  # :153-175
    s = lattice_system([5, 4, 3], 0.01, 1265.0)
    s.correction_matrices()
    s.set_material(5e4, 0.45, 1265.0, "neo_hookean")
    rng = np.random.RandomState(7)
    s.set("F", np.eye(3) + rng.uniform(-0.02, 0.02, (s.n, 3, 3)))
    s.momentum_rhs()
    a, m = s.get("a"), s.get("m")
    assert np.linalg.norm((m[:, None] * a).sum(0)) <= 1e-10 * (m * np.linalg.norm(a, axis=1)).sum()


def test_momentum_bruteforce_linear_kirchhoff():  # :177-203
    s = lattice_system([6, 6], 0.02, 1000.0)
    s.correction_matrices()
    s.set_material(1e5, 0.3, 1000.0, "linear")
    rng = np.random.RandomState(11)
    F = np.eye(2) + rng.uniform(-0.03, 0.03, (s.n, 2, 2))
    s.set("F", F)
    s.momentum_rhs()
    P = np.array([f @ O.second_pk(f, 1e5, 0.3, 1000.0, "linear") for f in F])
    ref = oracle_momentum_accel(s.get("r0"), s.get("V0"), s.get("m"), s.get("B0"), P, s.h)
    got = s.get("a")
    assert np.all(np.linalg.norm(got - ref, axis=1) <= 1e-12 * (1 + np.linalg.norm(ref, axis=1)))


def test_verlet_exact_for_constant_body_force():  # :205-224
    s = O.OracleSystem(np.zeros((1, 3)), 1.0, 1.0, 1.0, build=False)
    s.set_neighborhood([0, 0], np.zeros(0), np.zeros(0), np.zeros((0, 3)), np.zeros(0), np.zeros(0))
    s.set_material(1e5, 0.3, 1.0, "linear")
    s.set("body", [[0.0, -9.8, 0.0]])
    v0 = np.array([0.2, 0.1, 0.0])
    s.set("v", [v0])
    dt = 1e-3
    s.verlet_step(dt)
    g = np.array([0.0, -9.8, 0.0])
    assert np.linalg.norm(s.get("v")[0] - (v0 + dt * g)) <= 1e-15
    assert np.linalg.norm(s.get("r")[0] - (dt * v0 + 0.5 * dt * dt * g)) <= 1e-15


def test_verlet_rest_state_unchanged():  # :226-238
    s = lattice_system([5, 5], 0.01, 1000.0)
    s.correction_matrices()
    s.set_material(1e5, 0.3, 1000.0, "linear")
    r = s.get("r")
    s.verlet_step(1e-4)
    assert np.array_equal(s.get("r"), r)
    assert np.all(s.get("v") == 0.0)


def test_two_column_strip_conserves_momentum():  # :240-271
    dp = 0.01
    r0 = np.array([[ix * dp, iy * dp] for iy in range(3) for ix in range(2)])
    s = O.OracleSystem(r0, dp * dp, 1000.0, 1.3 * dp)
    s.set("v", np.array([[0.05 if ix == 0 else -0.05, 0.0] for iy in range(3) for ix in range(2)]))
    s.correction_matrices()
    s.set_material(1e5, 0.3, 1000.0, "linear")
    s.momentum_rhs()
    s.deformation_rate()
    m = s.get("m")
    p0 = total_momentum(m, s.get("v"))
    scale = momentum_scale(m, s.get("v"))
    for _ in range(1000):
        s.verlet_step(2e-5)
    assert np.linalg.norm(total_momentum(m, s.get("v")) - p0) <= 1e-12 * scale


def test_stable_dt_coarse_cantilever():  # :273-294
    dp = 0.04 / 6.0
    s = lattice_system([3, 3, 3], dp, 1265.0)
    s.set_material(5e4, 0.45, 1265.0, "neo_hookean")
    h = 1.3 * 0.04 / 6.0
    s.set("a", np.tile([0.0, -9.8, 0.0], (s.n, 1)))
    assert s.stable_dt(h) == approx(4.53e-4, 2e-3)
    s.set("a", np.zeros((s.n, 3)))
    c = O.material(5e4, 0.45, 1265.0)["c"]
    assert s.stable_dt(h) == approx(0.6 * h / c, 1e-12)


# ------------------------------------------------------------------ kernel / material / lattice
def test_kernel_normalisation_and_gradient():  # test_kernel.cpp
    for dim in (2, 3):
        for h in (1.0, 0.0086667):
            R = 2 * h
            n = 20000
            r = np.linspace(0, R, n + 1)
            w = np.array([O.kernel_value(h, dim, x) for x in r])
            shell = w * (2 * np.pi * r if dim == 2 else 4 * np.pi * r * r)
            simpson = (shell[0] + shell[-1] + 4 * shell[1:-1:2].sum() + 2 * shell[2:-1:2].sum()) * (R / n) / 3
            assert simpson == approx(1.0, 1e-4)
        k = 0.013
        assert O.kernel_value(k, dim, 2 * k) == 0.0 and O.grad_mag(k, dim, 2 * k) == 0.0
        for x in np.linspace(0.05, 1.9, 12) * k:
            fd = (O.kernel_value(k, dim, x + 1e-9 * k) - O.kernel_value(k, dim, x - 1e-9 * k)) / (2e-9 * k)
            assert O.grad_mag(k, dim, x) == pytest.approx(fd, rel=1e-6, abs=1e-6 * abs(fd) + 1e-3)
    assert O.kernel_value(1.0, 2, 0.0) == approx(7.0 / (4.0 * math.pi), 1e-12)


def test_material_constants():  # test_state.cpp:35-59
    m = O.material(5.0e4, 0.45, 1265.0)
    assert m["mu"] == approx(1.7241e4, 1e-4)
    assert m["lambda"] == approx(1.5517e5, 1e-4)
    assert m["K"] == approx(5.0e4 / (3.0 * (1.0 - 0.9)), 1e-12)
    assert m["c"] == approx(11.48, 1e-3)
    m = O.material(2e6, 0.3, 1000.0)
    assert m["c"] == approx(40.8248, 1e-5)  # BASELINE material


def test_stress_reference_state_and_inversion():  # test_state.cpp:85-93, 147-153
    for model in ("neo_hookean", "linear"):
        assert np.all(O.second_pk(np.eye(3), 5e4, 0.45, 1265.0, model) == 0.0)
    F = np.eye(3)
    F[0, 0] = -1.0
    with pytest.raises(O.OracleError):
        O.second_pk(F, 5e4, 0.45, 1265.0)


def test_box_lattice_counts():  # test_cases.cpp:10-31
    dp = 0.04 / 6.0
    r0 = O.box_lattice([0.0, -0.02, -0.02], [0.1, 0.02, 0.02], dp)
    assert len(r0) == 15 * 6 * 6
    assert len(O.box_lattice([0.0, 0.0], [0.1, 0.01], 0.01)) == 10
    with pytest.raises(O.OracleError):
        O.box_lattice([0.0, 0.0], [0.1, 0.001], 0.01)
    # same arithmetic as the fixture walk
    assert np.array_equal(O.box_lattice([0.0, 0.0], [0.04, 0.03], 0.01), lattice_r0([4, 3], 0.01))


def test_oracle_resumed_run_equals_uninterrupted():
    """The oracle loop continued across calls (orc_run resume: same RandomSource stream, t, step
    count) equals one uninterrupted run bit for bit (bench.py times steps W..W+K this way)."""
    from paper_2103_08932_b200 import scenarios as S
    cfg = S.cfg1(scale=4)
    out = []
    for split in (None, 7):
        o = O.OracleSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"], constrained=cfg["constrained"])
        o.set_material(S.E_MOD, S.NU, S.RHO0)
        o.set("v", cfg["v0"])
        o.set("body", cfg["body"])
        o.prepare()
        if split is None:
            r = o.run(eta=cfg["eta"], alpha=0.5, steps=20, seed=3)
        else:
            o.run(eta=cfg["eta"], alpha=0.5, steps=split, seed=3)
            r = o.run(eta=cfg["eta"], alpha=0.5, steps=20, seed=3, resume=True)
        out.append((r["steps"], r["damped"], r["t"], o.get("v"), o.get("r")))
    a, b = out
    assert a[:3] == b[:3] and a[0] == 20 and a[1] > 0
    assert np.array_equal(a[3], b[3]) and np.array_equal(a[4], b[4])
