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

Full step (``run_loop``). A slab advances only its own particles through the TL-SPH passes
(tlsph_dev_set_task_range also sets the ownership mask); its halo columns are refreshed from
their owners twice per step -- the (P B0, V0) record after pass A, which pass B gathers, and the
velocities after pass B's kick, which pass C and the sweep read -- and stable_dt's |v|max,
|a|max are combined across slabs (max is exact, so dt is bitwise that of one GPU). The
random-choice stream is replicated (RandomSource(seed) on every rank). With these, every
owned particle follows bit for bit the undivided device loop (DevSystem::run,
runner.cpp:341-391).

The driver is independent of the engine and the transport: an engine runs a slab's passes
and colour phases and packs/unpacks halo columns (``DeviceSlabEngine`` over a
``DeviceSystem``); a group moves the columns -- ``LocalGroup`` between slabs held by this
process with direct copies (the sequential statement of the protocol), ``DistGroup`` through
``torch.distributed`` point-to-point operations (NCCL between GPUs, gloo on CPU) with
all-reduces for the step scalars. ``sweep_in_process`` and ``SlabSweep`` are the sweep alone
over those two groups.
"""
from __future__ import annotations

import math
import os
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


def lattice_slab(lo, hi, dp, h, world, rank):
    """decompose() for a box lattice (generate_box_lattice, cases.cpp:21-46) without building the
    whole body: the global grid and column counts follow from the lattice axes, and only this
    rank's held particles are generated (reference order, x fastest). Returns (grid, ranges, slab,
    r0 of the held particles); identical to decompose() on the full lattice."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    if not (dp > 0.0) or np.any(hi - lo < dp * (1.0 - 1e-12)):
        raise ValueError("degenerate lattice")
    counts = []
    for d in range(len(lo)):
        q = (hi[d] - lo[d]) / dp
        counts.append(max(1, int(math.floor(q + 0.5))))
    axes = [lo[d] + (np.arange(counts[d], dtype=np.float64) + 0.5) * dp for d in range(len(lo))]
    cutoff = 2.0 * float(h)
    origin = np.array([a.min() for a in axes])
    dims = [max(1, int(math.floor((axes[d].max() - axes[d].min()) / cutoff)) + 1) for d in range(len(lo))]
    col_layer = np.clip(np.floor((axes[0] - origin[0]) / cutoff).astype(np.int64), 0, dims[0] - 1)
    per_layer = int(np.prod(counts[1:]))
    ranges = plan(np.bincount(col_layer, minlength=dims[0]) * per_layer, world)
    x0, x1 = ranges[rank]
    lo_col, hi_col = held_columns(x0, x1, dims[0])
    layers = np.nonzero((col_layer >= lo_col) & (col_layer < hi_col))[0]
    rest = np.meshgrid(*[axes[d] for d in range(len(lo) - 1, 0, -1)], indexing="ij")  # slowest first
    rest = [g.reshape(-1) for g in rest][::-1]  # axis 1 .. D-1, axis 1 fastest
    m = len(rest[0])
    r0 = np.empty((m * len(layers), len(lo)))
    r0[:, 0] = np.tile(axes[0][layers], m)
    for d in range(1, len(lo)):
        r0[:, d] = np.repeat(rest[d - 1], len(layers))
    ids = (np.arange(m)[:, None] * counts[0] + layers[None, :]).reshape(-1)
    return (origin, dims, cutoff), ranges, Slab(rank, x0, x1, ids), r0


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


def halo_transfers(ranges):
    """Owner-to-holder transfers that refresh every halo column: at each boundary the left
    slab's last own column (x1 - 1) goes right and the right slab's first (x1) goes left."""
    out = []
    for r in range(len(ranges) - 1):
        x1 = ranges[r][1]
        out.append(Transfer(x1 - 1, r, r + 1))
        out.append(Transfer(x1, r + 1, r))
    return out


class DeviceSlabEngine:
    """Passes, phases and halo-column buffers of one DeviceSystem slab (CUDA torch tensors)."""

    def __init__(self, system, dim, device="cuda"):
        self.d = system
        self.dim = dim
        self.device = device

    def phase(self, scheme, eta_tilde, dt, p, index):
        self.d.damping_phase(scheme, eta_tilde, dt, p, index)

    def verlet_pass(self, material, dt, p):
        self.d.verlet_pass(material, dt, p)

    def reduce(self, want_ke, check_step):
        return self.d.reduce_state(want_ke, check_step)

    def empty(self, x, field="velocity"):
        import torch

        w = self.d.column_width(field)
        return torch.empty(w * self.d.column_count(x), dtype=torch.float64, device=self.device)

    def pack(self, x, field="velocity"):
        buf = self.empty(x, field)
        if buf.numel():
            self.d.pack_column(x, buf.data_ptr(), field)
        return buf

    def unpack(self, x, buf, field="velocity"):
        import torch

        if buf.numel():
            torch.cuda.synchronize(self.device)  # a received buffer is written on the communicator's stream
            self.d.unpack_column(x, buf.data_ptr(), field)


class LocalGroup:
    """Slabs held by this process (one per GPU, or several on one): direct column copies."""

    def __init__(self, engines, ranges):
        self.engines = list(engines)
        self.ranges = list(ranges)

    def each(self, fn):
        for e in self.engines:
            fn(e)

    def exchange(self, transfers, field="velocity"):
        for t in transfers:
            self.engines[t.dst].unpack(t.column, self.engines[t.src].pack(t.column, field), field)

    def reduce(self, want_ke, check_step):
        vals = [e.reduce(want_ke, check_step) for e in self.engines]
        return max(v[0] for v in vals), max(v[1] for v in vals), sum(v[2] for v in vals)


class DistGroup:
    """This rank's slab; columns travel through torch.distributed point-to-point operations
    (NCCL between GPUs, gloo on CPU), step scalars through all-reduces."""

    def __init__(self, engine, ranges, rank):
        self.e = engine
        self.ranges = list(ranges)
        self.rank = rank

    def each(self, fn):
        fn(self.e)

    def exchange(self, transfers, field="velocity"):
        import torch.distributed as dist

        ops, unpack = [], []
        for t in transfers:
            if t.src == self.rank:
                ops.append(dist.P2POp(dist.isend, self.e.pack(t.column, field), t.dst))
            elif t.dst == self.rank:
                buf = self.e.empty(t.column, field)
                ops.append(dist.P2POp(dist.irecv, buf, t.src))
                unpack.append((t.column, buf))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for col, buf in unpack:
            self.e.unpack(col, buf, field)

    def reduce(self, want_ke, check_step):
        import torch
        import torch.distributed as dist

        vm, am, ke = self.e.reduce(want_ke, check_step)
        mx = torch.tensor([vm, am], dtype=torch.float64, device=self.e.device)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        if want_ke:
            s = torch.tensor([ke], dtype=torch.float64, device=self.e.device)
            dist.all_reduce(s, op=dist.ReduceOp.SUM)
            ke = float(s[0])
        return float(mx[0]), float(mx[1]), ke


def sweep(group, scheme, eta_tilde, dt, dim):
    """strang_damping_sweep (damping.cpp:125-182) over the slabs of a group: each colour phase
    on every slab, then that phase's column transfers."""
    if eta_tilde == 0.0:
        return
    for p, index, rx in colour_schedule(dim):
        group.each(lambda e: e.phase(scheme, eta_tilde, dt, p, index))
        group.exchange(phase_transfers(group.ranges, rx), "velocity")


def sweep_in_process(engines, ranges, scheme, eta_tilde, dt, dim):
    """One strang_damping_sweep over slab engines held by this process: every phase on every
    slab, then the phase's column transfers as direct copies (the protocol, sequentially)."""
    sweep(LocalGroup(engines, ranges), scheme, eta_tilde, dt, dim)


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


def sweep_linked(systems, scheme, eta_tilde, dt, count=1):
    """The fused sweep with the phase barrier on the devices: all phases of all slabs enqueued at
    once, each slab's stream waiting on its neighbours' previous-phase events
    (tlsph_dev_sweep_linked); no host synchronisation until the last phase. Returns the device
    time in seconds."""
    from paper_2103_08932_b200 import dev

    if eta_tilde == 0.0:
        return 0.0
    return dev.sweep_linked(systems, scheme, eta_tilde, dt, count)


class PhaseCounters:
    """Per-slab counts of enqueued colour phases, shared by the processes of one job through a file
    in /dev/shm (each process writes only its own slot). Before a process enqueues phase g with a
    wait on its neighbours' phase g-1 events, their counters must show g: cudaStreamWaitEvent binds
    to the event's most recent record at call time."""

    def __init__(self, path, world, create):
        import numpy as np

        mode = "w+" if create else "r+"
        self.path = path
        self.c = np.memmap(path, dtype=np.int64, mode=mode, shape=(world,))
        if create:
            self.c[:] = 0
            self.c.flush()

    def set(self, rank, value):
        self.c[rank] = value

    def wait(self, ranks, value, timeout=60.0):
        import time

        t0 = time.perf_counter()
        while any(int(self.c[r]) < value for r in ranks):
            if time.perf_counter() - t0 > timeout:
                raise TimeoutError(f"slab phase handshake: neighbours {ranks} did not reach phase {value}")

    def close(self, unlink):
        del self.c
        if unlink:
            try:
                os.unlink(self.path)
            except OSError:
                pass


class IpcSlabSweep:
    """One process's slab of a decomposed sweep, fused with its neighbours across processes
    (one process per GPU, e.g. under torchrun): the neighbours' velocity arrays are mapped through
    CUDA IPC, so each phase kernel stores the shared columns straight into them (over NVLink between
    GPUs), and the per-phase barrier is a stream wait on the neighbours' IPC phase events -- no host
    synchronisation between phases, only a host-side counter handshake that keeps every wait bound
    to the intended phase. `group`: torch.distributed process group for the one-time exchange of
    exports and cell tables (default group if None)."""

    def __init__(self, system, rank, world, group=None):
        import uuid

        import torch.distributed as dist

        self.d, self.rank, self.world = system, rank, world
        blob = system.ipc_export()
        cell_start = system.grid()["cell_start"]
        items = [None] * world
        dist.all_gather_object(items, (blob, cell_start), group=group)
        token = [uuid.uuid4().hex if rank == 0 else None]
        dist.broadcast_object_list(token, src=0, group=group)
        path = os.path.join("/dev/shm", f"tlsph_slab_{token[0]}")
        if rank == 0:
            self.counters = PhaseCounters(path, world, create=True)
            self.halo_counters = PhaseCounters(path + "_halo", world, create=True)
        dist.barrier(group=group)
        if rank != 0:
            self.counters = PhaseCounters(path, world, create=False)
            self.halo_counters = PhaseCounters(path + "_halo", world, create=False)
        dist.barrier(group=group)
        self.pushed = 0
        self.neighbours = [r for r in (rank - 1, rank + 1) if 0 <= r < world]
        if rank > 0:
            system.link_peer_ipc(0, *items[rank - 1])
        if rank + 1 < world:
            system.link_peer_ipc(1, *items[rank + 1])
        dist.barrier(group=group)  # every slab linked before any phase runs
        self.enqueued = 0
        self.nphase = 2 * 3 ** system.dim
        self._group = group

    def sweep(self, scheme, eta_tilde, dt, count=1):
        """`count` sweeps, enqueued phase by phase; returns after this slab's last phase ran and
        every neighbour store into this slab landed.

        Ordering at the ends of the call: the first phase stores into the neighbours' shared
        columns, so it waits on their marks (recorded after everything they enqueued before this
        sweep, e.g. verlet pass C reading those velocities); the last phase of a neighbour may
        still store into our owned boundary column, so the stream waits on its final phase event
        before the call returns (the next step's reductions read those velocities)."""
        if eta_tilde == 0.0:
            return
        self._barrier_mark()
        for k in range(count):
            for q in range(self.nphase):
                g = self.enqueued
                first = k == 0 and q == 0
                if not first:
                    self.counters.wait(self.neighbours, g)
                # the first phase is ordered by the marks; every later one by the neighbours'
                # previous phase (phase 0 of a later sweep: their last phase)
                self.d.sweep_phase_ipc(scheme, eta_tilde, dt, q, -1 if first else (q - 1) % self.nphase)
                self.enqueued = g + 1
                self.counters.set(self.rank, self.enqueued)
        self.counters.wait(self.neighbours, self.enqueued)
        self.d.wait_phase_ipc(self.nphase - 1)
        self.d.synchronize()

    def _barrier_mark(self):
        """Data-free cross-process ordering point: this slab's stream waits on the neighbours'
        work enqueued so far (shares the halo counter sequence: every rank issues the same
        sequence of halo pushes and marks)."""
        self.d.mark_ipc()
        self.pushed += 1
        self.halo_counters.set(self.rank, self.pushed)
        self.halo_counters.wait(self.neighbours, self.pushed)
        self.d.wait_mark_ipc()

    def halo(self, field):
        """The full loop's halo refresh across processes: push this slab's owned boundary columns of
        `field` into the neighbours, then (once they have pushed theirs) wait for their pushes on
        this slab's stream. No host synchronisation."""
        self.d.push_halo_ipc(field)
        self.pushed += 1
        self.halo_counters.set(self.rank, self.pushed)
        self.halo_counters.wait(self.neighbours, self.pushed)
        self.d.wait_halo_ipc(field)

    def close(self):
        import torch.distributed as dist

        dist.barrier(group=self._group)
        self.counters.close(unlink=self.rank == 0)
        self.halo_counters.close(unlink=self.rank == 0)


class IpcGroup(DistGroup):
    """run_loop's group for one process per GPU with the fused exchange: halo refreshes through
    IpcSlabSweep.halo (peer stores + IPC events), step scalars through torch.distributed
    all-reduces; pair it with sweeper=ipc_sweep.sweep."""

    def __init__(self, engine, ranges, rank, ipc_sweep):
        super().__init__(engine, ranges, rank)
        self.ipc = ipc_sweep

    def exchange(self, transfers, field="velocity"):
        self.ipc.halo(field)

    def reduce(self, want_ke, check_step):
        import torch
        import torch.distributed as dist

        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        vm, am, ke = self.e.reduce(want_ke, check_step)
        mx = torch.tensor([vm, am], dtype=torch.float64, device=dev)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        if want_ke:
            t = torch.tensor([ke], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            ke = float(t[0])
        return float(mx[0]), float(mx[1]), ke


class SlabSweep:
    """One rank's share of the decomposed sweep; halo columns travel through torch.distributed
    point-to-point operations (NCCL between GPUs, gloo on CPU)."""

    def __init__(self, engine, ranges, rank, dim):
        self.group = DistGroup(engine, ranges, rank)
        self.dim = dim

    def sweep(self, scheme, eta_tilde, dt):
        sweep(self.group, scheme, eta_tilde, dt, self.dim)


@dataclass
class LoopSpec:
    """The inputs of DevSystem::run (tlsph_dev_loop_params) a slab loop uses: fixed step count."""
    material: object  # dev.Material (rho0, c)
    h: float
    eta: float
    alpha: float
    steps: int
    seed: int = 0
    scheme: str = "particle_split"
    fixed_dt: float = 0.0
    elastic: bool = True


def step_dt(spec, vmax, amax, dim):
    """dt of one step as k_step_begin forms it: the fixed dt, else stable_dt (integrator.cpp:
    154-169) capped by the implicit viscous bound (damping.cpp:12-27, runner.cpp:343-351)."""
    if spec.fixed_dt > 0.0:
        return spec.fixed_dt
    h = spec.h
    bound = h / (spec.material.c + vmax)
    if amax > 0.0:
        b2 = math.sqrt(h / amax)
        bound = b2 if b2 < bound else bound
    dt = 0.6 * bound
    if spec.eta > 0.0 and spec.scheme in ("particle_split", "explicit"):
        nu = spec.eta / (spec.alpha * spec.material.rho0)
        vb = (0.5 if spec.scheme == "explicit" else 50.0) * h * h / (nu * dim)
        dt = vb if vb < dt else dt
    return dt


def run_loop(group, spec, dim, sweeper=None):
    """runner.cpp:341-391 over the slabs of a group, step for step as DevSystem::run executes
    it: step_begin (finite check of the previous step, dt from the combined maxima), verlet
    passes A, B, C with the halo refreshes between them, the random-choice sweep. The slabs
    must be prepared (runner.cpp:306-312) after their task ranges are set. `sweeper(scheme,
    eta_tilde, dt)`, if given, runs the damped steps' sweeps instead of the group's per-phase
    exchange -- the fused forms (`sweep_linked` over peer-linked slabs, `IpcSlabSweep.sweep`),
    which leave the shared columns current on both sides as the exchange does."""
    from . import dev

    if spec.scheme not in ("particle_split", "pairwise_split"):
        raise ValueError("slab loops sweep the split schemes only")
    damping = spec.eta > 0.0
    if damping and not (0.0 < spec.alpha <= 1.0):
        raise ValueError(f"random-choice probability must lie in (0, 1], got {spec.alpha}")
    # RandomSource(seed), one draw per step (damping.hpp:41-50, runner.cpp:358-360): replicated
    flags = dev.random_uniforms(spec.seed, spec.steps) < spec.alpha if damping else np.zeros(spec.steps, bool)
    eta_tilde = spec.eta / spec.alpha if damping else 0.0
    halo = halo_transfers(group.ranges)
    t, dt = 0.0, 0.0
    for k in range(spec.steps):
        vmax, amax, _ = group.reduce(False, k if k > 0 else -1)
        dt = step_dt(spec, vmax, amax, dim)
        if spec.elastic:
            group.each(lambda e: e.verlet_pass(spec.material, dt, 0))
            group.exchange(halo, "stress")
            group.each(lambda e: e.verlet_pass(spec.material, dt, 1))
            group.exchange(halo, "velocity")
            group.each(lambda e: e.verlet_pass(spec.material, dt, 2))
        if flags[k]:
            if sweeper is not None:
                sweeper(spec.scheme, eta_tilde, dt)
            else:
                sweep(group, spec.scheme, eta_tilde, dt, dim)
        t = t + dt
    group.reduce(False, spec.steps)  # check_finite of the last step
    return {"steps": spec.steps, "damped": int(flags.sum()), "t": t, "last_dt": dt}


# ---------------------------------------------------------------- the C entry point (csrc/cuda/group.cu)
class TorchComm:
    """tlsph_group_comm over torch.distributed (a gloo group: the collectives carry host bytes and
    scalars); keep the object alive while the C group uses it."""

    def __init__(self, group=None):
        import torch.distributed as dist

        from . import dev

        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self._ag = dev.ALLGATHER_FN(self._allgather)
        self._ar = dev.ALLREDUCE_FN(self._allreduce)
        self.struct = dev.GroupComm(None, self.rank, self.size, self._ag, self._ar)

    def _allgather(self, ctx, send, nbytes, recv):
        import ctypes as C

        import torch
        import torch.distributed as dist

        try:
            mine = torch.frombuffer(bytearray(C.string_at(send, nbytes)), dtype=torch.uint8) if nbytes else \
                torch.empty(0, dtype=torch.uint8)
            out = torch.empty(self.size * nbytes, dtype=torch.uint8)
            dist.all_gather_into_tensor(out, mine, group=self.group)
            if nbytes:
                C.memmove(recv, out.numpy().ctypes.data, self.size * nbytes)
            return 0
        except Exception:  # reported to the library as a failed collective
            return 1

    def _allreduce(self, ctx, values, count, op):
        import ctypes as C

        import numpy as np
        import torch
        import torch.distributed as dist

        try:
            arr = np.ctypeslib.as_array(values, shape=(count,))
            t = torch.from_numpy(arr.copy())
            dist.all_reduce(t, op=dist.ReduceOp.MAX if op == 0 else dist.ReduceOp.SUM, group=self.group)
            arr[:] = t.numpy()
            return 0
        except Exception:
            return 1


class CGroup:
    """tlsph_dev_group_* (C ABI) over this process's slab: the IPC-fused group loop and sweeps."""

    def __init__(self, system, comm):
        import ctypes as C

        from . import dev

        self.d, self.comm = system, comm
        self._h = C.c_void_p()
        st = dev.lib().tlsph_dev_group_create(system._h, C.byref(comm.struct), C.byref(self._h))
        if st != 0:
            raise dev.TlsphError(st, dev.lib().tlsph_group_last_error().decode())

    def _check(self, st):
        from . import dev

        if st != 0:
            raise dev.TlsphError(st, dev.lib().tlsph_group_last_error().decode())

    def sweep(self, scheme, eta_tilde, dt, count=1):
        from . import dev

        self._check(dev.lib().tlsph_dev_group_sweep(self._h, dev.SCHEMES[scheme], eta_tilde, dt, count))

    def run(self, material, *, h, eta, alpha, steps, seed=0, scheme="particle_split", fixed_dt=0.0, elastic=True):
        import ctypes as C

        from . import dev

        p = dev.LoopParams(material, h, eta, alpha, dev.SCHEMES[scheme], seed, 0.0, steps, fixed_dt,
                           1 if elastic else 0, 0, 1e-8, -1, 0.0, None, 0, 0, 0)
        r = dev.LoopResult()
        self._check(dev.lib().tlsph_dev_group_run(self._h, C.byref(p), C.byref(r)))
        return {"steps": r.steps, "damped": r.damped_steps, "t": r.t, "last_dt": r.last_dt,
                "device_s": r.total_seconds, "kernel_launches": int(r.kernel_launches)}

    def close(self):
        from . import dev

        if self._h:
            dev.lib().tlsph_dev_group_destroy(self._h)
            self._h = None


def plan_c(column_counts, world, min_width=2):
    """slabs.plan through the C ABI (tlsph_group_plan)."""
    import ctypes as C

    from . import dev

    counts = np.ascontiguousarray(column_counts, dtype=np.int64)
    out = (C.c_int * (2 * world))()
    if dev.lib().tlsph_group_plan(counts.ctypes.data_as(C.POINTER(C.c_int64)), len(counts), world, min_width, out) != 0:
        raise ValueError("no plan")
    return [(out[2 * r], out[2 * r + 1]) for r in range(world)]
