"""X-slab decomposition of the colour-scheduled damping sweep over ranks.

The body's global cell grid is the reference's (``build_cell_grid``, neighbors.cpp:24-59:
origin = min r0, cell = cutoff = 2h, dims = floor(extent / cutoff) + 1). Rank r owns the
cells whose x lies in ``[x0, x1)`` -- those are its sweep tasks -- and holds the particles of
the columns ``[x0 - 1, x1 + 1)`` (one halo column each side), numbered in ascending
reference id. Because every slab is binned in the *global* grid, cell indices, colours and
the in-cell order are those of the undivided body, so each phase performs exactly the
reference's updates and the result is bitwise that of one GPU (neighbors.hpp:50-52:
same-colour stencils are disjoint, so reordering cells within a colour is bit-neutral).

Exchange. In a phase with x-residue ``rx`` a cell column ``c`` is written by the tasks at
``t`` with ``t = rx (mod 3)`` and ``|t - c| <= 1`` -- exactly one task column, hence exactly
one rank. Across the boundary between ``x1 - 1`` (rank r) and ``x1`` (rank r + 1) both
columns are therefore written every phase, each by one side, and the writer sends the
whole column to the other side after the phase (``phase_transfers``). Slabs are at least
two columns wide so a rank's tasks never reach past its neighbour's halo.

The fused form (``link_peers`` / ``sweep_fused``): each slab's phase kernels store the shared
columns straight into the neighbouring slab's arrays (NVLink peer access between GPUs), so the
only inter-slab operation left is the per-phase ordering.

The driver is independent of the engine and the transport: an engine runs a slab's colour
phases and packs/unpacks halo columns (``DeviceSlabEngine`` over a ``DeviceSystem``);
``SlabSweep`` exchanges the columns through ``torch.distributed`` (NCCL between GPUs, gloo
on CPU) and ``sweep_in_process`` runs several slabs in one process with direct copies (the
sequential statement of the same protocol).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def global_grid(r0, h):
    """(origin, dims, cell) of build_cell_grid (neighbors.cpp:24-59) for reference positions r0."""
    r0 = np.asarray(r0, dtype=np.float64)
    cutoff = 2.0 * float(h)
    lo, hi = r0.min(axis=0), r0.max(axis=0)
    dims = [max(1, int(math.floor((hi[d] - lo[d]) / cutoff)) + 1) for d in range(r0.shape[1])]
    return lo.copy(), dims, cutoff


def cell_columns(r0, origin, cell, dims0):
    """Cell x index of every particle (CellGrid::coords_of_position, clamped)."""
    x = np.floor((np.asarray(r0)[:, 0] - origin[0]) / cell).astype(np.int64)
    return np.clip(x, 0, dims0 - 1)


def plan(column_counts, world, min_width=2):
    """Contiguous cell-column ranges [(x0, x1), ...], one per rank, balanced by particle count."""
    counts = np.asarray(column_counts, dtype=np.int64)
    ncol = len(counts)
    if world < 1:
        raise ValueError("world size must be positive")
    if ncol < min_width * world:
        raise ValueError(f"{ncol} cell columns cannot give {world} slabs of width >= {min_width}")
    cum = np.concatenate([[0], np.cumsum(counts)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        x = int(np.searchsorted(cum, target, side="left"))
        # keep every slab at least min_width wide on both sides of the cut
        x = max(x, cuts[-1] + min_width)
        x = min(x, ncol - min_width * (world - r))
        cuts.append(x)
    cuts.append(ncol)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def held_columns(x0, x1, dims0):
    """Columns a slab holds: owned plus one halo column each side."""
    return max(0, x0 - 1), min(dims0, x1 + 1)


def local_ids(columns, x0, x1, dims0):
    """Ascending reference ids of the particles a slab holds."""
    lo, hi = held_columns(x0, x1, dims0)
    return np.nonzero((columns >= lo) & (columns < hi))[0]


def colour_schedule(dim):
    """The 2 x 3^D phases of strang_damping_sweep in order: (pass, index, x-residue).

    Colour b's residues are (b % 3, b // 3 % 3, b // 9) with x fastest; the forward pass runs
    b = index, the reverse pass b = 3^D - 1 - index (damping.cpp:125-182)."""
    nb = 3 ** dim
    out = []
    for p in (0, 1):
        for index in range(nb):
            b = index if p == 0 else nb - 1 - index
            out.append((p, index, b % 3))
    return out


def _writes(task_lo, task_hi, column, rx):
    """True when a task column t in [task_lo, task_hi) with t = rx (mod 3) writes `column`."""
    return any(task_lo <= t < task_hi and t % 3 == rx for t in (column - 1, column, column + 1))


@dataclass
class Transfer:
    column: int
    src: int  # rank that wrote the column this phase
    dst: int  # rank that holds it as owner or halo


def phase_transfers(ranges, rx):
    """Column transfers after a phase with x-residue rx, for slab ranges [(x0, x1), ...]."""
    out = []
    for r in range(len(ranges) - 1):
        (a0, a1), (b0, b1) = ranges[r], ranges[r + 1]
        for col in (a1 - 1, a1):
            left, right = _writes(a0, a1, col, rx), _writes(b0, b1, col, rx)
            if left and right:
                raise AssertionError("two writers of one column in a phase")  # disjoint stencils
            if left:
                out.append(Transfer(col, r, r + 1))
            elif right:
                out.append(Transfer(col, r + 1, r))
    return out


@dataclass
class Slab:
    rank: int
    x0: int
    x1: int
    ids: np.ndarray  # reference ids held, ascending


def decompose(r0, h, world):
    """Global grid and one Slab per rank for reference positions r0."""
    origin, dims, cell = global_grid(r0, h)
    cols = cell_columns(r0, origin, cell, dims[0])
    ranges = plan(np.bincount(cols, minlength=dims[0]), world)
    slabs = [Slab(r, x0, x1, local_ids(cols, x0, x1, dims[0])) for r, (x0, x1) in enumerate(ranges)]
    return (origin, dims, cell), slabs


def make_device_slab(grid, slab, r0, V0, rho0, h, constrained=None):
    """DeviceSystem of one slab: the held particles binned in the global grid, tasks = owned columns."""
    from . import dev

    ids = slab.ids
    n = len(r0)
    V0 = np.broadcast_to(np.asarray(V0, dtype=np.float64), (n,))
    rho0 = np.broadcast_to(np.asarray(rho0, dtype=np.float64), (n,))
    cons = None if constrained is None else np.asarray(constrained)[ids]
    d = dev.DeviceSystem(np.asarray(r0)[ids], V0[ids], rho0[ids], h, cons, grid=grid[:2])
    d.set_task_range(slab.x0, slab.x1)
    return d


class DeviceSlabEngine:
    """Phase runner + halo-column buffers of one DeviceSystem slab (CUDA torch tensors)."""

    def __init__(self, system, dim, device="cuda"):
        self.d = system
        self.dim = dim
        self.device = device

    def phase(self, scheme, eta_tilde, dt, p, index):
        self.d.damping_phase(scheme, eta_tilde, dt, p, index)

    def empty(self, x):
        import torch

        return torch.empty(self.dim * self.d.column_count(x), dtype=torch.float64, device=self.device)

    def pack(self, x):
        buf = self.empty(x)
        if buf.numel():
            self.d.pack_column(x, buf.data_ptr())
        return buf

    def unpack(self, x, buf):
        import torch

        if buf.numel():
            torch.cuda.synchronize(self.device)  # a received buffer is written on the communicator's stream
            self.d.unpack_column(x, buf.data_ptr())


def sweep_in_process(engines, ranges, scheme, eta_tilde, dt, dim):
    """One strang_damping_sweep over slab engines held by this process: every phase on every
    slab, then the phase's column transfers as direct copies (the protocol, sequentially)."""
    if eta_tilde == 0.0:
        return
    for p, index, rx in colour_schedule(dim):
        for e in engines:
            e.phase(scheme, eta_tilde, dt, p, index)
        for t in phase_transfers(ranges, rx):
            engines[t.dst].unpack(t.column, engines[t.src].pack(t.column))


def link_peers(systems):
    """Fused form of the exchange: each slab's phase kernels store the columns it shares with its
    x-neighbours straight into their arrays (tlsph_dev_link_peer; NVLink peer access across GPUs)."""
    for r in range(len(systems) - 1):
        systems[r].link_peer(1, systems[r + 1])
        systems[r + 1].link_peer(0, systems[r])


def sweep_fused(systems, scheme, eta_tilde, dt, dim):
    """One strang_damping_sweep over peer-linked slabs held by this process (one per GPU or all on
    one): the phases of all slabs, then the next phase; the exchange happens inside the kernels."""
    if eta_tilde == 0.0:
        return
    for p, index, _ in colour_schedule(dim):
        for d in systems:  # each call returns after its kernel: the phase barrier
            d.damping_phase(scheme, eta_tilde, dt, p, index)


class SlabSweep:
    """One rank's share of the decomposed sweep; halo columns travel through torch.distributed
    point-to-point operations (NCCL between GPUs, gloo on CPU)."""

    def __init__(self, engine, ranges, rank, dim):
        self.e = engine
        self.ranges = list(ranges)
        self.rank = rank
        self.dim = dim

    def sweep(self, scheme, eta_tilde, dt):
        import torch.distributed as dist

        if eta_tilde == 0.0:
            return
        for p, index, rx in colour_schedule(self.dim):
            self.e.phase(scheme, eta_tilde, dt, p, index)
            ops, unpack = [], []
            for t in phase_transfers(self.ranges, rx):
                if t.src == self.rank:
                    ops.append(dist.P2POp(dist.isend, self.e.pack(t.column), t.dst))
                elif t.dst == self.rank:
                    buf = self.e.empty(t.column)
                    ops.append(dist.P2POp(dist.irecv, buf, t.src))
                    unpack.append((t.column, buf))
            if ops:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
            for col, buf in unpack:
                self.e.unpack(col, buf)
