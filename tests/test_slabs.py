"""x-slab decomposition of the damping sweep (paper_2103_08932_b200/slabs.py).

CPU: the partition and exchange protocol, run with the oracle as the per-slab engine, both
in one process and as a world-size-2/3 gloo job; the decomposed sweep must equal the
undivided oracle sweep bit for bit (same-colour stencils are disjoint, neighbors.hpp:50-52).
GPU: the same protocol over DeviceSystem slabs (tlsph_dev_create_in_grid + per-phase
sweeps + column pack/unpack) against the undivided device sweep, bit for bit.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

from tests.fixtures import lattice_r0, random_velocities
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

    def empty(self, x):
        return torch.empty(self.dim * len(self._column(x)), dtype=torch.float64)

    def pack(self, x):
        return torch.from_numpy(np.ascontiguousarray(self.o.get("v")[self._column(x)].T).ravel().copy())

    def unpack(self, x, buf):
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
        assert np.array_equal(vv[own], ref[s.ids[own]])


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
        assert np.array_equal(vv[own], ref[s.ids[own]])
        # halo columns hold the neighbours' current values too
        assert np.array_equal(vv, ref[s.ids])


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
