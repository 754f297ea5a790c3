"""x-slab decomposition of the damping sweep and the full step (SURVEY.md §8(e),
paper_2103_08932_b200/slabs.py).

CPU: the partition and exchange protocol, run with the oracle as the per-slab engine, both
in one process and as a world-size-2/3 gloo job; the decomposed sweep must equal the
undivided oracle sweep bit for bit (same-colour stencils are disjoint, neighbors.hpp:50-52).
The full-step loop (halo refreshes between the TL-SPH passes, combined step scalars) runs
over a column-coupled toy engine under gloo and must equal the undivided toy run.
GPU: the same protocols over DeviceSystem slabs (tlsph_dev_create_in_grid + per-phase
sweeps + column pack/unpack, verlet passes on owned particles) against the undivided device
sweep and the undivided device loop (tlsph_dev_run), bit for bit.
"""
from __future__ import annotations

import math
import os
import types
import socket

import numpy as np
import pytest
import torch

from tests.fixtures import assert_slab_field, lattice_r0, random_velocities
from paper_2103_08932_b200 import slabs

import oracle.oracle as orc

DP, RHO, H = 0.01, 1000.0, 0.013


def body(dim, counts=None, clamp=True):
    counts = counts or ([26, 7] if dim == 2 else [17, 5, 4])
    r0 = lattice_r0(counts, DP)
    cons = (r0[:, 0] < 0.02).astype(np.uint8) if clamp else np.zeros(len(r0), np.uint8)
    v = random_velocities(len(r0), dim, 1.0, 5)
    v[cons == 1] = 0.0
    return r0, cons, v


class OracleSlab:
    """Slab engine over the CPU oracle: the held particles, the owned rows of the global
    neighbourhood, and the reference cell loop restricted to the owned columns."""

    def __init__(self, glob, slab, r0, cons, v):
        self.g = glob
        self.slab = slab
        self.dim = r0.shape[1]
        ids = slab.ids
        self.lmap = np.full(len(r0), -1, dtype=np.int64)
        self.lmap[ids] = np.arange(len(ids))
        self.cons = cons
        self.o = orc.OracleSystem(r0[ids], DP ** self.dim, RHO, H, cons[ids], build=False)
        nb = glob["nbh"]
        cols = glob["cols"]
        off = [0]
        parts = {k: [] for k in ("neighbor", "r0_len", "e0", "dwdr0", "pair_factor")}
        for g in ids:
            if slab.x0 <= cols[g] < slab.x1:
                s0, s1 = nb["offsets"][g], nb["offsets"][g + 1]
                js = self.lmap[nb["neighbor"][s0:s1]]
                assert (js >= 0).all(), "owned row reaches past the halo"
                parts["neighbor"].append(js)
                for k in ("r0_len", "e0", "dwdr0", "pair_factor"):
                    parts[k].append(nb[k][s0:s1])
                off.append(off[-1] + (s1 - s0))
            else:
                off.append(off[-1])
        cat = {k: (np.concatenate(a) if a else np.zeros((0, self.dim) if k == "e0" else 0)) for k, a in parts.items()}
        self.o.set_neighborhood(np.array(off), cat["neighbor"], cat["r0_len"], cat["e0"], cat["dwdr0"],
                                cat["pair_factor"])
        self.o.set("v", v[ids])

    def phase(self, scheme, eta, dt, p, index):
        assert scheme == "particle_split"
        nb = 3 ** self.dim
        b = index if p == 0 else nb - 1 - index
        g = self.g
        for cell in g["blocks"][b]:
            if not (self.slab.x0 <= cell % g["dims"][0] < self.slab.x1):
                continue
            ps = g["cell_particles"][g["cell_start"][cell]:g["cell_start"][cell + 1]]
            for i in (ps if p == 0 else ps[::-1]):
                if not self.cons[i]:
                    self.o.particle_split_update(int(self.lmap[i]), eta, 0.5 * dt)

    def _column(self, x):
        g = self.g
        d0 = g["dims"][0]
        out = []
        for q in range((len(g["cell_start"]) - 1) // d0):
            c = q * d0 + x
            out.extend(g["cell_particles"][g["cell_start"][c]:g["cell_start"][c + 1]])
        return self.lmap[np.array(out, dtype=np.int64)]

    def empty(self, x, field="velocity"):
        return torch.empty(self.dim * len(self._column(x)), dtype=torch.float64)

    def pack(self, x, field="velocity"):
        return torch.from_numpy(np.ascontiguousarray(self.o.get("v")[self._column(x)].T).ravel().copy())

    def unpack(self, x, buf, field="velocity"):
        v = self.o.get("v")
        v[self._column(x)] = buf.numpy().reshape(self.dim, -1).T
        self.o.set("v", v)

    def owned(self):
        """(reference ids, velocities) of the owned particles."""
        cols = self.g["cols"]
        keep = (cols[self.slab.ids] >= self.slab.x0) & (cols[self.slab.ids] < self.slab.x1)
        return self.slab.ids[keep], self.o.get("v")[keep]


def global_oracle(r0, cons, v):
    o = orc.OracleSystem(r0, DP ** r0.shape[1], RHO, H, cons)
    o.set("v", v)
    gr = o.grid()
    origin, dims, cell = slabs.global_grid(r0, H)
    assert np.allclose(origin, gr["origin"]) and list(dims) == list(gr["dims"]) and cell == gr["cell_size"]
    glob = {"nbh": o.neighborhood(), "blocks": o.blocks(), "dims": gr["dims"], "cell_start": gr["cell_start"],
            "cell_particles": gr["cell_particles"], "cols": slabs.cell_columns(r0, origin, cell, dims[0])}
    return o, glob


# ---------------------------------------------------------------- partition / protocol logic
def test_plan_balanced_and_wide_enough():
    counts = np.array([5, 9, 9, 9, 9, 9, 9, 9, 9, 9, 9, 4])
    for world in (1, 2, 3, 4, 6):
        ranges = slabs.plan(counts, world)
        assert ranges[0][0] == 0 and ranges[-1][1] == len(counts)
        assert all(a1 == b0 for (_, a1), (b0, _) in zip(ranges, ranges[1:]))
        assert all(x1 - x0 >= 2 for x0, x1 in ranges)
    with pytest.raises(ValueError):
        slabs.plan(counts, 7)


@pytest.mark.parametrize("dim", [2, 3])
def test_every_boundary_column_has_one_writer_per_phase(dim):
    ranges = [(0, 4), (4, 6), (6, 11), (11, 14)]
    for p, index, rx in slabs.colour_schedule(dim):
        ts = slabs.phase_transfers(ranges, rx)
        # both columns of every boundary travel every phase, from the side whose task wrote them
        assert sorted(t.column for t in ts) == sorted(c for (_, x1) in ranges[:-1] for c in (x1 - 1, x1))
        for t in ts:
            src_lo, src_hi = ranges[t.src]
            writers = [x for x in range(src_lo, src_hi) if x % 3 == rx and abs(x - t.column) <= 1]
            assert len(writers) == 1


def test_schedule_matches_sweep_order():
    sched = slabs.colour_schedule(3)
    assert len(sched) == 54
    assert [s[1] for s in sched[:27]] == list(range(27)) and sched[27] == (1, 0, 26 % 3)


# ---------------------------------------------------------------- oracle engine, in process
@pytest.mark.parametrize("dim,world", [(2, 2), (2, 3), (3, 2), (3, 3)])
def test_decomposed_sweep_equals_undivided_oracle(dim, world):
    r0, cons, v = body(dim)
    o, glob = global_oracle(r0, cons, v)
    grid, parts = slabs.decompose(r0, H, world)
    engines = [OracleSlab(glob, s, r0, cons, v) for s in parts]
    ranges = [(s.x0, s.x1) for s in parts]
    for _ in range(2):
        o.damping_sweep("particle_split", 160.0, 1e-4)
        slabs.sweep_in_process(engines, ranges, "particle_split", 160.0, 1e-4, dim)
    ref = o.get("v")
    got = np.empty_like(ref)
    seen = np.zeros(len(r0), bool)
    for e in engines:
        ids, vv = e.owned()
        got[ids] = vv
        seen[ids] = True
    assert seen.all()
    assert np.array_equal(got, ref)


# ---------------------------------------------------------------- gloo, world size 2 and 3
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_rank(rank, world, port, dim, result_dir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r0, cons, v = body(dim)
        o, glob = global_oracle(r0, cons, v)
        grid, parts = slabs.decompose(r0, H, world)
        eng = OracleSlab(glob, parts[rank], r0, cons, v)
        sweep = slabs.SlabSweep(eng, [(s.x0, s.x1) for s in parts], rank, dim)
        for _ in range(2):
            sweep.sweep("particle_split", 160.0, 1e-4)
        ids, vv = eng.owned()
        np.save(os.path.join(result_dir, f"rank{rank}.npy"), np.concatenate([ids[:, None], vv], axis=1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_slab_sweep_equals_undivided_oracle(tmp_path, world):
    import torch.multiprocessing as mp

    dim = 3
    mp.spawn(_gloo_rank, args=(world, _free_port(), dim, str(tmp_path)), nprocs=world, join=True)
    r0, cons, v = body(dim)
    o, _ = global_oracle(r0, cons, v)
    for _ in range(2):
        o.damping_sweep("particle_split", 160.0, 1e-4)
    ref = o.get("v")
    got = np.full_like(ref, np.nan)
    for r in range(world):
        a = np.load(tmp_path / f"rank{r}.npy")
        got[a[:, 0].astype(np.int64)] = a[:, 1:]
    assert np.array_equal(got, ref)


# ---------------------------------------------------------------- GPU: DeviceSystem slabs
@pytest.mark.gpu
@pytest.mark.parametrize("dim,world,mode", [(2, 3, "ordered"), (3, 2, "ordered"), (3, 3, "fast")])
def test_device_slabs_equal_undivided_device(dim, world, mode):
    from paper_2103_08932_b200 import dev

    r0, cons, v = body(dim, [40, 9] if dim == 2 else [24, 6, 5])
    whole = dev.DeviceSystem(r0, DP ** dim, RHO, H, cons)
    whole.set_reduction(mode)
    whole.set("v", v)
    grid, parts = slabs.decompose(r0, H, world)
    systems = [slabs.make_device_slab(grid, s, r0, DP ** dim, RHO, H, cons) for s in parts]
    engines = []
    for s, d in zip(parts, systems):
        d.set_reduction(mode)
        d.set("v", v[s.ids])
        engines.append(slabs.DeviceSlabEngine(d, dim))
    ranges = [(s.x0, s.x1) for s in parts]
    for _ in range(3):
        whole.damping_sweep("particle_split", 160.0, 1e-4)
        slabs.sweep_in_process(engines, ranges, "particle_split", 160.0, 1e-4, dim)
    ref = whole.get("v")
    cols = slabs.cell_columns(r0, grid[0], grid[2], grid[1][0])
    for s, d in zip(parts, systems):
        vv = d.get("v")
        own = (cols[s.ids] >= s.x0) & (cols[s.ids] < s.x1)
        assert_slab_field(vv[own], ref[s.ids[own]], mode)


@pytest.mark.gpu
@pytest.mark.parametrize("dim,world,mode", [(2, 3, "ordered"), (3, 2, "fast"), (3, 3, "ordered"),
                                            (3, 3, "fast")])
def test_fused_peer_slabs_equal_undivided_device(dim, world, mode):
    """Fused exchange: phase kernels store shared columns into the neighbouring slab directly."""
    from paper_2103_08932_b200 import dev

    r0, cons, v = body(dim, [40, 9] if dim == 2 else [24, 6, 5])
    whole = dev.DeviceSystem(r0, DP ** dim, RHO, H, cons)
    whole.set_reduction(mode)
    whole.set("v", v)
    grid, parts = slabs.decompose(r0, H, world)
    systems = [slabs.make_device_slab(grid, s, r0, DP ** dim, RHO, H, cons) for s in parts]
    for s, d in zip(parts, systems):
        d.set_reduction(mode)
        d.set("v", v[s.ids])
    slabs.link_peers(systems)
    for _ in range(3):
        whole.damping_sweep("particle_split", 160.0, 1e-4)
        slabs.sweep_fused(systems, "particle_split", 160.0, 1e-4, dim)
    ref = whole.get("v")
    cols = slabs.cell_columns(r0, grid[0], grid[2], grid[1][0])
    for s, d in zip(parts, systems):
        vv = d.get("v")
        own = (cols[s.ids] >= s.x0) & (cols[s.ids] < s.x1)
        assert_slab_field(vv[own], ref[s.ids[own]], mode)
        # halo columns hold the neighbours' current values too
        assert_slab_field(vv, ref[s.ids], mode)


@pytest.mark.gpu
@pytest.mark.parametrize("dim,world,mode,scheme", [(2, 3, "ordered", "particle_split"), (3, 2, "fast", "particle_split"),
                                                   (3, 4, "ordered", "particle_split"), (3, 3, "fast", "particle_split"),
                                                   (3, 3, "ordered", "pairwise_split"), (3, 2, "fast", "pairwise_split")])
def test_linked_slabs_equal_undivided_device(dim, world, mode, scheme):
    """Fused exchange with the per-phase barrier on the devices (stream event dependencies between
    neighbouring slabs, no host synchronisation): bitwise the undivided sweep."""
    from paper_2103_08932_b200 import dev

    r0, cons, v = body(dim, [40, 9] if dim == 2 else [30, 6, 5])
    whole = dev.DeviceSystem(r0, DP ** dim, RHO, H, cons)
    whole.set_reduction(mode)
    whole.set("v", v)
    grid, parts = slabs.decompose(r0, H, world)
    systems = [slabs.make_device_slab(grid, s, r0, DP ** dim, RHO, H, cons) for s in parts]
    for s, d in zip(parts, systems):
        d.set_reduction(mode)
        d.set("v", v[s.ids])
    slabs.link_peers(systems)
    whole.damping_sweep(scheme, 160.0, 1e-4, count=3)
    el = slabs.sweep_linked(systems, scheme, 160.0, 1e-4, count=3)
    assert el > 0.0
    ref = whole.get("v")
    for s, d in zip(parts, systems):
        assert_slab_field(d.get("v"), ref[s.ids], mode if scheme == "particle_split" else "ordered")


@pytest.mark.gpu
def test_device_phases_compose_to_sweep():
    from paper_2103_08932_b200 import dev

    r0, cons, v = body(3)
    a = dev.DeviceSystem(r0, DP ** 3, RHO, H, cons)
    b = dev.DeviceSystem(r0, DP ** 3, RHO, H, cons)
    for d in (a, b):
        d.set_reduction("ordered")
        d.set("v", v)
    a.damping_sweep("particle_split", 160.0, 1e-4)
    for p, index, _ in slabs.colour_schedule(3):
        b.damping_phase("particle_split", 160.0, 1e-4, p, index)
    assert np.array_equal(a.get("v"), b.get("v"))


# ---------------------------------------------------------------- full-step loop, toy engine (CPU)
class ToySlab:
    """Column-coupled stand-in for a slab with the dependency pattern of the real step: pass A
    writes a per-particle record from own state (v, and w as F from dF/dt), pass B reads the
    records of the x-neighbour columns and kicks v, pass C writes w from the velocities of the
    x-neighbour columns (it changes no velocity, like the real pass C); a sweep task writes its
    column and both x-neighbours. Undivided = one slab owning every column."""

    NCOL, M = 13, 3

    def __init__(self, x0, x1):
        self.x0, self.x1 = x0, x1
        self.lo, self.hi = max(0, x0 - 1), min(self.NCOL, x1 + 1)
        c = np.arange(self.NCOL)[:, None] + np.arange(self.M)[None, :] / self.M
        self.v = np.sin(1.7 * c)[self.lo:self.hi].copy()
        self.rec = np.zeros_like(self.v)
        self.a = np.zeros_like(self.v)
        self.w = np.zeros_like(self.v)
        self.device = "cpu"

    def _own(self):
        return range(self.x0 - self.lo, self.x1 - self.lo)

    def _get(self, c, arr):
        k = c - self.lo
        return arr[k] if 0 <= c < self.NCOL else 0.0

    def verlet_pass(self, mat, dt, p):
        new_v = self.v.copy()
        for k in self._own():
            c = k + self.lo
            if p == 0:
                self.rec[k] = np.cos(self.v[k]) + 0.25 * c + self.w[k]
            elif p == 1:
                self.a[k] = self._get(c - 1, self.rec) + self._get(c + 1, self.rec) - 2.0 * self.rec[k]
                new_v[k] = self.v[k] + dt * self.a[k]
            else:
                self.w[k] = self.w[k] + 0.3 * (self._get(c - 1, self.v) - self._get(c + 1, self.v))
        self.v = new_v

    def phase(self, scheme, eta, dt, p, index):
        b = index if p == 0 else 26 - index
        for t in range(self.x0, self.x1):
            if t % 3 != b % 3:
                continue
            cols = [c for c in (t - 1, t, t + 1) if 0 <= c < self.NCOL]
            s = sum(self.v[c - self.lo].sum() for c in cols)
            for c in cols:
                self.v[c - self.lo] = 0.9 * self.v[c - self.lo] + 0.1 * np.tanh(s + c) * eta * dt

    def reduce(self, want_ke, check_step):
        own = list(self._own())
        return (float(np.abs(self.v[own]).max()), float(np.abs(self.a[own]).max()),
                float(0.5 * (self.v[own] ** 2).sum()) if want_ke else 0.0)

    def _arr(self, field):
        return self.v if field == "velocity" else self.rec

    def empty(self, x, field="velocity"):
        return torch.empty(self.M, dtype=torch.float64)

    def pack(self, x, field="velocity"):
        return torch.from_numpy(self._arr(field)[x - self.lo].copy())

    def unpack(self, x, buf, field="velocity"):
        self._arr(field)[x - self.lo] = buf.numpy()

    def owned(self):
        return np.arange(self.x0, self.x1), self.v[list(self._own())]


TOY_SPEC = dict(material=types.SimpleNamespace(c=3.0, rho0=1.0), h=0.05, eta=0.4, alpha=0.5, steps=9, seed=4)


def _toy_reference():
    whole = ToySlab(0, ToySlab.NCOL)
    out = slabs.run_loop(slabs.LocalGroup([whole], [(0, ToySlab.NCOL)]), slabs.LoopSpec(**TOY_SPEC), 3)
    return whole.v, out


def test_toy_loop_in_process_equals_undivided():
    ref, out_ref = _toy_reference()
    ranges = slabs.plan(np.ones(ToySlab.NCOL), 3)
    engines = [ToySlab(a, b) for a, b in ranges]
    out = slabs.run_loop(slabs.LocalGroup(engines, ranges), slabs.LoopSpec(**TOY_SPEC), 3)
    assert out == out_ref and 0 < out["damped"] < out["steps"]
    got = np.concatenate([e.owned()[1] for e in engines])
    assert np.array_equal(got, ref)
    # without the halo refreshes the slabs drift from the undivided run
    saved = slabs.halo_transfers
    try:
        slabs.halo_transfers = lambda ranges: []
        engines = [ToySlab(a, b) for a, b in ranges]
        slabs.run_loop(slabs.LocalGroup(engines, ranges), slabs.LoopSpec(**TOY_SPEC), 3)
        assert not np.array_equal(np.concatenate([e.owned()[1] for e in engines]), ref)
    finally:
        slabs.halo_transfers = saved


def test_step_dt_matches_device_formula():
    mat = types.SimpleNamespace(c=40.0, rho0=1000.0)
    spec = slabs.LoopSpec(material=mat, h=0.013, eta=100.0, alpha=0.2, steps=1)
    dt = slabs.step_dt(spec, 0.5, 2.0e3, 3)
    acoustic = 0.6 * min(0.013 / (40.0 + 0.5), math.sqrt(0.013 / 2.0e3))
    visc = 50.0 * 0.013 * 0.013 / ((100.0 / (0.2 * 1000.0)) * 3)
    assert dt == min(acoustic, visc)
    assert slabs.step_dt(slabs.LoopSpec(material=mat, h=0.013, eta=0.0, alpha=1.0, steps=1), 0.5, 0.0, 3) == \
        0.6 * (0.013 / 40.5)
    assert slabs.step_dt(slabs.LoopSpec(material=mat, h=0.013, eta=1.0, alpha=1.0, steps=1, fixed_dt=1e-5),
                         9.0, 9.0, 3) == 1e-5


def _gloo_toy_rank(rank, world, port, result_dir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ranges = slabs.plan(np.ones(ToySlab.NCOL), world)
        eng = ToySlab(*ranges[rank])
        out = slabs.run_loop(slabs.DistGroup(eng, ranges, rank), slabs.LoopSpec(**TOY_SPEC), 3)
        ids, vv = eng.owned()
        np.save(os.path.join(result_dir, f"rank{rank}.npy"), np.concatenate([ids[:, None], vv], axis=1))
        np.save(os.path.join(result_dir, f"out{rank}.npy"), np.array([out["t"], out["damped"], out["last_dt"]]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_toy_loop_equals_undivided(tmp_path, world):
    import torch.multiprocessing as mp

    mp.spawn(_gloo_toy_rank, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    ref, out_ref = _toy_reference()
    got = np.full_like(ref, np.nan)
    for r in range(world):
        a = np.load(tmp_path / f"rank{r}.npy")
        got[a[:, 0].astype(np.int64)] = a[:, 1:]
        o = np.load(tmp_path / f"out{r}.npy")
        assert o[0] == out_ref["t"] and o[1] == out_ref["damped"] and o[2] == out_ref["last_dt"]
    assert np.array_equal(got, ref)


# ---------------------------------------------------------------- GPU: full step over device slabs
@pytest.mark.gpu
@pytest.mark.parametrize("dim,world,mode", [(2, 2, "ordered"), (2, 3, "fast"), (3, 2, "ordered"),
                                            (3, 3, "fast")])
@pytest.mark.parametrize("fused", [False, True])
def test_slab_loop_equals_undivided_device_loop(dim, world, mode, fused):
    """TL-SPH passes on owned particles + halo refreshes + decomposed random-choice sweeps
    reproduce tlsph_dev_run on the undivided body bit for bit (elastic, gravity, clamped root)."""
    from paper_2103_08932_b200 import dev, scenarios as S

    mat = S.material()
    r0, cons, v = body(dim, [40, 9] if dim == 2 else [24, 6, 5])
    v = 0.05 * v
    g = np.zeros_like(r0)
    g[:, 1] = -9.81
    eta = 0.2 * RHO * mat.c * H
    steps, alpha, seed = 14, 0.5, 3
    whole = dev.DeviceSystem(r0, DP ** dim, RHO, H, cons)
    whole.set_reduction(mode)
    whole.set("v", v)
    whole.set("body", g)
    whole.prepare(mat)
    ref = whole.run(mat, eta=eta, alpha=alpha, steps=steps, seed=seed)
    grid, parts = slabs.decompose(r0, H, world)
    engines = []
    for s in parts:
        d = slabs.make_device_slab(grid, s, r0, DP ** dim, RHO, H, cons)
        d.set_reduction(mode)
        d.set("v", v[s.ids])
        d.set("body", g[s.ids])
        d.prepare(mat)
        engines.append(slabs.DeviceSlabEngine(d, dim))
    sweeper = None
    if fused:  # damped steps through the linked sweep (peer stores, device-side phase barrier)
        systems = [e.d for e in engines]
        slabs.link_peers(systems)
        sweeper = lambda scheme, et, dt: slabs.sweep_linked(systems, scheme, et, dt)  # noqa: E731
    out = slabs.run_loop(slabs.LocalGroup(engines, [(s.x0, s.x1) for s in parts]),
                         slabs.LoopSpec(mat, H, eta, alpha, steps, seed=seed), dim, sweeper=sweeper)
    assert out["damped"] == ref["damped"] > 0
    if mode == "ordered":
        assert out["t"] == ref["t"] and out["last_dt"] == ref["last_dt"]
    else:  # FAST: the step size follows max |v|, |a| of fields equal to 1e-12 (assert_slab_field)
        assert math.isclose(out["t"], ref["t"], rel_tol=1e-12) and math.isclose(out["last_dt"], ref["last_dt"], rel_tol=1e-12)
    cols = slabs.cell_columns(r0, grid[0], grid[2], grid[1][0])
    for name in ("v", "r", "F", "dFdt", "rho", "a"):
        want = whole.get(name)
        for s, e in zip(parts, engines):
            own = (cols[s.ids] >= s.x0) & (cols[s.ids] < s.x1)
            assert_slab_field(e.d.get(name)[own], want[s.ids[own]], mode, name)


# ---------------------------------------------------------------- cross-process phase handshake
def _counter_rank(rank, world, port, result_dir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        path = os.path.join(result_dir, "counters")
        if rank == 0:
            c = slabs.PhaseCounters(path, world, create=True)
        dist.barrier()
        if rank != 0:
            c = slabs.PhaseCounters(path, world, create=False)
        dist.barrier()
        nb = [r for r in (rank - 1, rank + 1) if 0 <= r < world]
        seen = []
        for g in range(200):  # the IpcSlabSweep discipline: wait for the neighbours' phase g-1
            if g > 0:
                c.wait(nb, g, timeout=30.0)
                seen.append(min(int(c.c[r]) for r in nb))
            c.set(rank, g + 1)
        np.save(os.path.join(result_dir, f"seen{rank}.npy"), np.array(seen))
        dist.barrier()
        c.close(unlink=rank == 0)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_phase_counter_handshake(tmp_path, world):
    """Host side of the cross-process fused sweep: no rank ever runs more than one phase ahead of
    a neighbour, and the lockstep never deadlocks."""
    import torch.multiprocessing as mp

    mp.spawn(_counter_rank, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        seen = np.load(os.path.join(tmp_path, f"seen{r}.npy"))
        assert np.all(seen >= np.arange(1, 200)) and np.all(seen <= np.arange(1, 200) + 1)


def _ipc_rank(rank, world, port, dim, scheme, mode, result_dir):
    import torch.distributed as dist

    from paper_2103_08932_b200 import dev

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev.select_device(0)  # one GPU: every process's slab on device 0 (IPC within the device)
        r0, cons, v = body(dim, [30, 6, 5] if dim == 3 else [40, 9])
        grid, parts = slabs.decompose(r0, H, world)
        d = slabs.make_device_slab(grid, parts[rank], r0, DP ** dim, RHO, H, cons)
        d.set_reduction(mode)
        d.set("v", v[parts[rank].ids])
        sweep = slabs.IpcSlabSweep(d, rank, world)
        sweep.sweep(scheme, 160.0, 1e-4, count=2)
        sweep.sweep(scheme, 160.0, 1e-4, count=1)
        np.save(os.path.join(result_dir, f"v{rank}.npy"), d.get("v"))
        np.save(os.path.join(result_dir, f"ids{rank}.npy"), parts[rank].ids)
        sweep.close()
        del d
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("dim,world,mode,scheme", [(3, 2, "fast", "particle_split"), (3, 3, "ordered", "particle_split"),
                                                   (2, 3, "fast", "particle_split"), (3, 2, "fast", "pairwise_split")])
def test_ipc_slabs_equal_undivided_device(tmp_path, dim, world, mode, scheme):
    """One process per slab (all on GPU 0 here), fused exchange through CUDA IPC mappings and IPC
    phase events, host-side counter handshake: bitwise the undivided sweep."""
    import torch.multiprocessing as mp

    from paper_2103_08932_b200 import dev

    mp.spawn(_ipc_rank, args=(world, _free_port(), dim, scheme, mode, str(tmp_path)), nprocs=world, join=True)
    r0, cons, v = body(dim, [30, 6, 5] if dim == 3 else [40, 9])
    whole = dev.DeviceSystem(r0, DP ** dim, RHO, H, cons)
    whole.set_reduction(mode)
    whole.set("v", v)
    whole.damping_sweep(scheme, 160.0, 1e-4, count=3)
    ref = whole.get("v")
    for r in range(world):
        ids = np.load(os.path.join(tmp_path, f"ids{r}.npy"))
        assert_slab_field(np.load(os.path.join(tmp_path, f"v{r}.npy")), ref[ids],
                          mode if scheme == "particle_split" else "ordered")


def _ipc_loop_rank(rank, world, port, dim, mode, result_dir):
    import torch.distributed as dist

    from paper_2103_08932_b200 import dev, scenarios as S

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev.select_device(0)
        mat = S.material()
        r0, cons, v = body(dim, [40, 9] if dim == 2 else [24, 6, 5])
        v = 0.05 * v
        g = np.zeros_like(r0)
        g[:, 1] = -9.81
        grid, parts = slabs.decompose(r0, H, world)
        s = parts[rank]
        d = slabs.make_device_slab(grid, s, r0, DP ** dim, RHO, H, cons)
        d.set_reduction(mode)
        d.set("v", v[s.ids])
        d.set("body", g[s.ids])
        d.prepare(mat)
        ipc = slabs.IpcSlabSweep(d, rank, world)
        group = slabs.IpcGroup(slabs.DeviceSlabEngine(d, dim), [(p.x0, p.x1) for p in parts], rank, ipc)
        eta = 0.2 * RHO * mat.c * H
        out = slabs.run_loop(group, slabs.LoopSpec(mat, H, eta, 0.5, 14, seed=3), dim,
                             sweeper=lambda scheme, et, dt: ipc.sweep(scheme, et, dt))
        d.synchronize()
        np.savez(os.path.join(result_dir, f"r{rank}.npz"), ids=s.ids, x0=s.x0, x1=s.x1, t=out["t"],
                 damped=out["damped"], **{k: d.get(k) for k in ("v", "r", "F", "dFdt", "rho", "a")})
        ipc.close()
        del d
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("dim,world,mode", [(3, 2, "fast"), (3, 3, "ordered"), (2, 2, "ordered")])
def test_ipc_slab_loop_equals_undivided_device_loop(tmp_path, dim, world, mode):
    """One process per slab: the full TL-SPH + random-choice damping loop with halo pushes and sweeps
    through CUDA IPC (no host synchronisation inside a step besides the dt all-reduce): every owned
    particle's state equals the undivided device loop bit for bit."""
    import torch.multiprocessing as mp

    from paper_2103_08932_b200 import dev, scenarios as S

    mp.spawn(_ipc_loop_rank, args=(world, _free_port(), dim, mode, str(tmp_path)), nprocs=world, join=True)
    mat = S.material()
    r0, cons, v = body(dim, [40, 9] if dim == 2 else [24, 6, 5])
    v = 0.05 * v
    g = np.zeros_like(r0)
    g[:, 1] = -9.81
    whole = dev.DeviceSystem(r0, DP ** dim, RHO, H, cons)
    whole.set_reduction(mode)
    whole.set("v", v)
    whole.set("body", g)
    whole.prepare(mat)
    ref = whole.run(mat, eta=0.2 * RHO * mat.c * H, alpha=0.5, steps=14, seed=3)
    grid, parts = slabs.decompose(r0, H, world)
    cols = slabs.cell_columns(r0, grid[0], grid[2], grid[1][0])
    for r in range(world):
        z = np.load(os.path.join(tmp_path, f"r{r}.npz"))
        assert int(z["damped"]) == ref["damped"] > 0
        assert float(z["t"]) == ref["t"] if mode == "ordered" else math.isclose(float(z["t"]), ref["t"], rel_tol=1e-12)
        ids = z["ids"]
        own = (cols[ids] >= int(z["x0"])) & (cols[ids] < int(z["x1"]))
        for name in ("v", "r", "F", "dFdt", "rho", "a"):
            assert_slab_field(z[name][own], whole.get(name)[ids[own]], mode, (r, name))


@pytest.mark.parametrize("lo,hi,world", [([0, 0, 0], [0.4, 0.1, 0.08], 3), ([0, -0.2, -0.2], [0.8, 0.2, 0.2], 4),
                                         ([0, 0], [1.0, 0.1], 2)])
def test_lattice_slab_equals_decompose(lo, hi, world):
    """The per-rank lattice generator (no whole body on the host) reproduces decompose() exactly."""
    from paper_2103_08932_b200 import scenarios as S

    r0, _ = S.box_lattice(lo, hi, DP)
    grid, parts = slabs.decompose(r0, H, world)
    for r in range(world):
        g2, ranges, sl, lr0 = slabs.lattice_slab(lo, hi, DP, H, world, r)
        assert np.array_equal(g2[0], grid[0]) and g2[1] == grid[1] and g2[2] == grid[2]
        assert (sl.x0, sl.x1) == (parts[r].x0, parts[r].x1)
        assert np.array_equal(sl.ids, parts[r].ids) and np.array_equal(lr0, r0[parts[r].ids])



# ---------------------------------------------------------------- cross-process sweep ordering
class _RecordingSlab:
    """Stands in for a DeviceSystem slab in IpcSlabSweep: records the asynchronous calls."""

    def __init__(self, dim):
        self.dim = dim
        self.log = []

    def ipc_export(self):
        return b"x"

    def grid(self):
        return {"cell_start": np.zeros(2, np.int64)}

    def link_peer_ipc(self, side, blob, cell_start):
        self.log.append(("link", side))

    def sweep_phase_ipc(self, scheme, eta_tilde, dt, q, wait_q):
        self.log.append(("phase", q, wait_q))

    def mark_ipc(self):
        self.log.append(("mark",))

    def wait_mark_ipc(self):
        self.log.append(("wait_mark",))

    def wait_phase_ipc(self, q):
        self.log.append(("wait_phase", q))

    def push_halo_ipc(self, field):
        self.log.append(("push", field))

    def wait_halo_ipc(self, field):
        self.log.append(("wait_halo", field))

    def synchronize(self):
        self.log.append(("sync",))


def _ipc_order_rank(rank, world, port, result_dir):
    import pickle

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d = _RecordingSlab(3)
        sw = slabs.IpcSlabSweep(d, rank, world)
        sw.halo("stress")
        sw.halo("velocity")
        sw.sweep("particle_split", 1.0, 1e-5, count=2)
        sw.halo("stress")
        sw.sweep("particle_split", 1.0, 1e-5)
        sw.close()
        with open(os.path.join(result_dir, f"log{rank}.pkl"), "wb") as fh:
            pickle.dump(d.log, fh)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ipc_sweep_ordering_points(tmp_path, world):
    """IpcSlabSweep.sweep: every sweep call starts with a mark + wait on the
    neighbours' marks before its first phase (whose stores reach the neighbours' shared columns
    while they may still run verlet pass C), chains every later phase on the neighbours' previous
    phase, and ends with a wait on their last phase before the host synchronises."""
    import pickle

    import torch.multiprocessing as mp

    mp.spawn(_ipc_order_rank, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    nphase = 54
    for r in range(world):
        with open(os.path.join(tmp_path, f"log{r}.pkl"), "rb") as fh:
            log = [x for x in pickle.load(fh) if x[0] != "link"]
        calls = []
        i = 0
        while i < len(log):
            if log[i][0] == "mark":
                j = log.index(("sync",), i)
                calls.append(log[i:j + 1])
                i = j + 1
            else:
                i += 1
        assert [len(c) for c in calls] == [2 + 2 * nphase + 2, 2 + nphase + 2]
        for c, count in zip(calls, (2, 1)):
            assert c[:2] == [("mark",), ("wait_mark",)]
            phases = c[2:-2]
            assert phases[0] == ("phase", 0, -1)
            for g, p in enumerate(phases[1:], start=1):
                assert p == ("phase", g % nphase, (g - 1) % nphase)
            assert c[-2:] == [("wait_phase", nphase - 1), ("sync",)]


# ---------------------------------------------------------------- the C entry point (tlsph_dev_group_*)
def test_c_plan_equals_python_plan():
    """tlsph_group_plan (csrc/cuda/group.cu) is slabs.plan: random column populations, 1-8 ranks."""
    rng = np.random.RandomState(17)
    for _ in range(200):
        ncol = int(rng.randint(2, 120))
        world = int(rng.randint(1, max(2, min(8, ncol // 2) + 1)))
        counts = rng.randint(0, 5000, ncol)
        if rng.rand() < 0.3:
            counts[rng.rand(ncol) < 0.5] = 0
        assert slabs.plan_c(counts, world) == slabs.plan(counts, world), (counts.tolist(), world)
    with pytest.raises(ValueError):
        slabs.plan_c(np.ones(3), 2)


def test_c_step_dt_equals_python_step_dt_bitwise():
    """The group loop's dt (tlsph_group_step_dt, k_step_begin's formula) equals slabs.step_dt bit for
    bit: with and without |a|max, fixed dt, each scheme's viscous bound."""
    import ctypes as C

    from paper_2103_08932_b200 import dev, scenarios as S

    mat = S.material()
    rng = np.random.RandomState(5)
    for scheme in ("particle_split", "pairwise_split", "explicit"):
        for _ in range(300):
            h = float(rng.uniform(1e-3, 5e-2))
            eta = float(rng.choice([0.0, rng.uniform(1.0, 500.0)]))
            alpha = float(rng.uniform(0.05, 1.0))
            fixed = float(rng.choice([0.0, 0.0, 1e-4]))
            vmax, amax = float(rng.exponential(0.5)), float(rng.choice([0.0, rng.exponential(50.0)]))
            dim = int(rng.choice([2, 3]))
            spec = slabs.LoopSpec(mat, h, eta, alpha, 1, scheme=scheme, fixed_dt=fixed)
            p = dev.LoopParams(mat, h, eta, alpha, dev.SCHEMES[scheme], 0, 0.0, 1, fixed, 1, 0, 1e-8, -1, 0.0, None,
                               0, 0, 0)
            got = dev.lib().tlsph_group_step_dt(C.byref(p), dim, vmax, amax)
            assert got == slabs.step_dt(spec, vmax, amax, dim), (scheme, h, eta, alpha, fixed, vmax, amax, dim)


def _comm_selftest_rank(rank, world, port, result_dir):
    import torch.distributed as dist

    from paper_2103_08932_b200 import dev

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ctypes as C

        comm = slabs.TorchComm()
        st = dev.lib().tlsph_group_comm_selftest(C.byref(comm.struct))
        msg = dev.lib().tlsph_group_last_error().decode()
        np.save(os.path.join(result_dir, f"st{rank}.npy"), np.array([st]))
        assert st == 0, msg
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_c_group_communicator_over_gloo(tmp_path, world):
    """The C group's collectives (tlsph_group_comm) carried by torch.distributed gloo across
    processes on the CPU: allgather in rank order, max / sum all-reduces (tlsph_group_comm_selftest)."""
    import torch.multiprocessing as mp

    mp.spawn(_comm_selftest_rank, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert int(np.load(os.path.join(tmp_path, f"st{r}.npy"))[0]) == 0


def _c_group_loop_rank(rank, world, port, dim, mode, result_dir):
    import torch.distributed as dist

    from paper_2103_08932_b200 import dev, scenarios as S

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev.select_device(0)
        mat = S.material()
        r0, cons, v = body(dim, [40, 9] if dim == 2 else [24, 6, 5])
        v = 0.05 * v
        g = np.zeros_like(r0)
        g[:, 1] = -9.81
        grid, parts = slabs.decompose(r0, H, world)
        s = parts[rank]
        d = slabs.make_device_slab(grid, s, r0, DP ** dim, RHO, H, cons)
        d.set_reduction(mode)
        d.set("v", v[s.ids])
        d.set("body", g[s.ids])
        d.prepare(mat)
        grp = slabs.CGroup(d, slabs.TorchComm())
        out = grp.run(mat, h=H, eta=0.2 * RHO * mat.c * H, alpha=0.5, steps=14, seed=3)
        grp.sweep("particle_split", 160.0, 1e-4, count=2)
        d.synchronize()
        np.savez(os.path.join(result_dir, f"r{rank}.npz"), ids=s.ids, x0=s.x0, x1=s.x1, t=out["t"],
                 damped=out["damped"], **{k: d.get(k) for k in ("v", "r", "F", "dFdt", "rho", "a")})
        grp.close()
        del d
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("dim,world,mode", [(3, 2, "fast"), (3, 3, "ordered"), (2, 2, "ordered")])
def test_c_group_loop_equals_undivided_device_loop(tmp_path, dim, world, mode):
    """tlsph_dev_group_run + tlsph_dev_group_sweep (the C entry point; one process per slab, gloo
    carrying the set-up and dt scalars, CUDA IPC the halo and colour-phase stores): every owned
    particle equals the undivided device loop followed by two sweeps, bit for bit."""
    import torch.multiprocessing as mp

    from paper_2103_08932_b200 import dev, scenarios as S

    mp.spawn(_c_group_loop_rank, args=(world, _free_port(), dim, mode, str(tmp_path)), nprocs=world, join=True)
    mat = S.material()
    r0, cons, v = body(dim, [40, 9] if dim == 2 else [24, 6, 5])
    v = 0.05 * v
    g = np.zeros_like(r0)
    g[:, 1] = -9.81
    whole = dev.DeviceSystem(r0, DP ** dim, RHO, H, cons)
    whole.set_reduction(mode)
    whole.set("v", v)
    whole.set("body", g)
    whole.prepare(mat)
    ref = whole.run(mat, eta=0.2 * RHO * mat.c * H, alpha=0.5, steps=14, seed=3)
    whole.damping_sweep("particle_split", 160.0, 1e-4, count=2)
    grid, parts = slabs.decompose(r0, H, world)
    cols = slabs.cell_columns(r0, grid[0], grid[2], grid[1][0])
    for r in range(world):
        z = np.load(os.path.join(tmp_path, f"r{r}.npz"))
        assert int(z["damped"]) == ref["damped"] > 0
        assert float(z["t"]) == ref["t"] if mode == "ordered" else math.isclose(float(z["t"]), ref["t"], rel_tol=1e-12)
        ids = z["ids"]
        own = (cols[ids] >= int(z["x0"])) & (cols[ids] < int(z["x1"]))
        for name in ("v", "r", "F", "dFdt", "rho", "a"):
            assert_slab_field(z[name][own], whole.get(name)[ids[own]], mode, (r, name))
