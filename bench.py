#!/usr/bin/env python3
"""Benchmark of the B200 hot path (BASELINE.json metric), one JSON line on rank 0.

Workload (default, the config BASELINE's metric is quoted on that fits one GPU):
  cfg2 — 3D damping-only sweep, 64^3 = 262,144 particles, fp64, 27-colour
  particle-split Strang sweep, alpha = 1, fixed dt = 0.6 h / c.
  One "step" = one full damping sweep (forward + mirrored reverse pass).
  metric = damping pair-updates per second (DPU/s): 2 * S_free per sweep.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2|cfg1|cfg3]
  python bench.py --impl reference ...   # the reference CPU path (oracle port, all host cores)

Multi-GPU (torchrun, one rank per GPU): every rank runs its own cfg2 body for the
headline `value` (replicas of the 64^3 block, so per-GPU work matches N = 1), timed
with CUDA events on the library's stream, max over ranks; value = total DPU / max time.
The line adds `sweep_sharded`: BASELINE cfg5's weak scaling, one x-slab of an
N x 250-layer body per rank with the fused cross-process exchange (slabs.IpcSlabSweep);
at N = 1 `sweep_at_scale` times the same per-GPU body undivided.
Other legs: `particle_steps` (cfg3 full loop, PS/s), `parity` (500 cfg2 sweeps vs the
oracle), `cpu_baseline` (oracle port on the host cores).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}
BYTES_SLOT = 12          # neighbor i32 + pair_factor f64
P_D = {3: 65, 2: 49}     # v r/w + m + flag + offset per free particle per half-pass
P_S = {3: 1091, 2: 587}  # per particle-step minimal traffic


def load_traffic():
    """DRAM bytes per launch of the sweep phase from the committed ncu --set full capture (profiles/)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return float(json.load(fh)["dram_bytes_per_launch"])
    except Exception:
        return None


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return PEAKS_FALLBACK["hbm_gbs"], "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled during the timed region: NVML every
    few milliseconds (nvidia-ml-py), nvidia-smi as the fallback."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0, period=0.002):
        self.index = index
        self.period = period
        self.samples = []  # (sm_mhz, max_mhz, set of reasons)
        self._stop = threading.Event()
        self._t = None

    def _nvml(self):
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            bits = get_reasons(h)
            self.samples.append((float(sm), float(mx), {k for k, b in self.REASONS.items() if bits & b}))
            self._stop.wait(self.period)

    def _smi(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                f = [x.strip() for x in out.stdout.strip().split(",")]
                names = list(self.REASONS)
                self.samples.append((float(f[0]), float(f[1]),
                                     {names[k] for k in range(4) if f[2 + k].lower().startswith("active")}))
            except Exception:
                pass
            self._stop.wait(0.2)

    def _run(self):
        try:
            self._nvml()
        except Exception:
            self._smi()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.05)  # first sample before the timed region starts
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        sm = [x[0] for x in self.samples]
        reasons = set()
        for x in self.samples:
            reasons |= x[2]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": self.samples[-1][1] if self.samples else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def barrier_and_max(value, ws):
    if ws == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def cuda_sync():
    try:
        import torch
        if torch.cuda.is_available():
            torch.cuda.synchronize()
    except Exception:
        pass


# ----------------------------------------------------------------------------- cfg2 (headline)
def free_slots(off, cons):
    if cons is None:
        return int(off[-1]), len(off) - 1
    counts = off[1:] - off[:-1]
    free = cons == 0
    return int(counts[free].sum()), int(free.sum())


def cpu_sweep_sample(cfg, threads, budget_s, min_sweeps=1):
    """Times full oracle sweeps (the reference CPU path, OpenMP over same-colour cells) within a budget."""
    from oracle import oracle as O
    o = O.OracleSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"], constrained=cfg["constrained"])
    o.set("v", cfg["v0"])
    eta_t = cfg["eta"] / cfg["alpha"]
    o.damping_sweep("particle_split", eta_t, cfg["fixed_dt"], threads=threads)  # warm
    times = []
    t_start = time.perf_counter()
    while len(times) < min_sweeps or (time.perf_counter() - t_start) < budget_s:
        t0 = time.perf_counter()
        o.damping_sweep("particle_split", eta_t, cfg["fixed_dt"], threads=threads)
        times.append(time.perf_counter() - t0)
        if len(times) >= 1000:
            break
    return times, o


def run_cfg2(args, ws, rank):
    from paper_2103_08932_b200 import dev
    from paper_2103_08932_b200 import scenarios as S
    cfg = S.cfg2()
    d = S.build_device(cfg, prepare=False)
    offsets = d.row_offsets()
    s_free, n_free = free_slots(offsets, cfg["constrained"])
    dpu_per_sweep = 2 * s_free
    b_sweep = 2 * (BYTES_SLOT * s_free + P_D[3] * n_free)
    eta_t = cfg["eta"] / cfg["alpha"]
    dt = cfg["fixed_dt"]
    # warmup
    for _ in range(args.warmup):
        d.damping_sweep("particle_split", eta_t, dt)
    barrier(ws)
    cuda_sync()
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        elapsed = d.damping_sweep("particle_split", eta_t, dt, count=args.steps)  # CUDA events on the stream
    cuda_sync()
    barrier(ws)
    t_max = barrier_and_max(elapsed, ws)
    value = dpu_per_sweep * args.steps * ws / t_max
    phase_launches = 54
    avg_launch = elapsed / (args.steps * phase_launches)
    achieved = (b_sweep / phase_launches) / avg_launch / 1e9
    peak, peak_src = load_peaks()

    # e2e through the C ABI with host buffers: v host->device, sweep, v device->host, every step,
    # from / into pinned host memory
    import numpy as np
    import torch
    v_in = torch.empty(cfg["v0"].shape, dtype=torch.float64, pin_memory=True).numpy()
    v_out = torch.empty(cfg["v0"].shape, dtype=torch.float64, pin_memory=True).numpy()
    v_in[...] = cfg["v0"]
    h2d = d2h = v_in.nbytes
    d.set("v", v_in)
    d.damping_sweep("particle_split", eta_t, dt)
    d.get("v", out=v_out)
    barrier(ws)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        d.set("v", v_in)
        d.damping_sweep("particle_split", eta_t, dt)
        d.get("v", out=v_out)
    t_e2e = barrier_and_max(time.perf_counter() - t0, ws)
    e2e = dpu_per_sweep * args.steps * ws / t_e2e

    out = {
        "metric": "damping pair-updates/s (fp64 particle-split Strang sweep)",
        "value": value,
        "unit": "DPU/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_max / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded 64^3 lattice, v ~ N(0,1) Box-Muller from RandomSource(1))",
        "config": {"workload": "cfg2: 3D damping-only sweep, 64^3 lattice, 27-colour particle-split, alpha=1",
                   "particles": int(d.n), "slots": int(offsets[-1]), "dpu_per_step": dpu_per_sweep,
                   "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                   "l2": "inputs larger than L2 (CSR 200 MB + 20 MB state > 126 MB L2); no flush",
                   "reduction": "fast (warp-shuffle)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": load_traffic(), "kernel": "k_sweep_fast (one colour phase)",
                     "bytes_per_launch": b_sweep / phase_launches, "avg_launch_s": avg_launch,
                     "peak_source": peak_src},
        "e2e": {"value": e2e, "unit": "DPU/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": "tlsph_dev_set_field(V) + tlsph_dev_damping_sweep + tlsph_dev_get_field(V), host buffers"},
        "gpu_launches": phase_launches * args.steps,
        "clocks": clk.summary(),
    }
    if rank == 0 and ws == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        from oracle import oracle as O
        threads = min(threads, O.openmp_threads())
        times, _ = cpu_sweep_sample(cfg, threads, budget_s=args.cpu_budget)
        t_cpu = statistics.median(times)
        times1, _ = cpu_sweep_sample(cfg, 1, budget_s=min(args.cpu_budget, 5.0))
        out["cpu_baseline"] = {"value": dpu_per_sweep / t_cpu, "unit": "DPU/s", "cores": threads, "kind": "port",
                               "sample": f"{len(times)} full cfg2 sweeps (median), oracle OpenMP over same-colour cells",
                               "value_1_thread": dpu_per_sweep / statistics.median(times1),
                               "sample_1_thread": f"{len(times1)} full cfg2 sweeps (median), 1 thread"}
        if args.parity_sweeps > 0:
            out["parity"] = cfg2_parity(cfg, d, args.parity_sweeps, threads)
    return out


def cfg2_parity(cfg, d, sweeps, threads):
    """BASELINE cfg2's check: velocity-variance decay over `sweeps` sweeps from v0, GPU (FAST) against
    the oracle (reference arithmetic), plus the relative L2 distance of the final velocity fields."""
    import numpy as np
    from oracle import oracle as O
    eta_t, dt = cfg["eta"] / cfg["alpha"], cfg["fixed_dt"]
    d.set("v", cfg["v0"])
    d.damping_sweep("particle_split", eta_t, dt, count=sweeps)
    vg = d.get("v")
    o = O.OracleSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"], constrained=cfg["constrained"])
    o.set("v", cfg["v0"])
    for _ in range(sweeps):
        o.damping_sweep("particle_split", eta_t, dt, threads=threads)
    vo = o.get("v")
    var0 = float(np.var(cfg["v0"]))
    return {"sweeps": sweeps, "var_v0": var0, "var_gpu": float(np.var(vg)), "var_oracle": float(np.var(vo)),
            "rel_l2_v": float(np.linalg.norm(vg - vo) / np.linalg.norm(vo)), "tolerance": 1e-10,
            "mode": "fast (warp-shuffle reductions) vs oracle"}


def particle_steps(args, ws, rank):
    """Second half of BASELINE.json's metric: particle-steps/s of the full device-resident loop
    (TL-SPH step + random-choice splitting damping, runner.cpp:341-391) on cfg3, the 3D cantilever
    beam (640,000 particles), FAST reductions; the reference CPU path (oracle port, OpenMP) timed on
    a bounded sample of the same loop."""
    from paper_2103_08932_b200 import scenarios as S
    cfg = S.cfg3()
    steps = max(50, min(args.ps_steps, 2000))
    d = S.build_device(cfg, prepare=True)
    d.set_reduction("fast")
    r = d.run(S.material(), eta=cfg["eta"], alpha=cfg["alpha"], steps=steps, seed=cfg["seed"])
    t_max = barrier_and_max(r["total_s"], ws)
    n = int(d.n)
    slots = int(d.slot_count)
    # B_step = S*2*(4+8+8D) + N*P_s (+ B_sweep on damped steps), P_s = 1,091 B (3D)
    b_elastic = slots * 2 * (4 + 8 + 8 * 3) + n * 1091
    t_el = r["elastic_s"] / max(r["steps"], 1)
    peak, peak_src = load_peaks()
    out = {"metric": "particle-steps/s (fp64 TL-SPH step + splitting damping, random choice)",
           "value": n * r["steps"] * ws / t_max, "unit": "PS/s", "steps": r["steps"], "damped_steps": r["damped"],
           "ms_per_step": t_max / max(r["steps"], 1) * 1e3, "elastic_ms_per_step": t_el * 1e3,
           "damping_ms_per_damped_step": r["damping_s"] / max(r["damped"], 1) * 1e3,
           "config": {"workload": "cfg3: 3D cantilever beam 400x40x40, neo-Hookean, gravity, 5-layer clamp, "
                                  "alpha=0.2", "particles": n, "slots": slots, "reduction": "fast"},
           "roofline": {"bound": "hbm", "kernel": "TL-SPH step (passes A-C + step-begin reduction)",
                        "achieved": b_elastic / t_el / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": b_elastic / t_el / 1e9 / peak, "bytes_per_step": b_elastic, "peak_source": peak_src}}
    if rank == 0 and ws == 1 and not args.no_cpu:
        from oracle import oracle as O
        out["cpu_baseline"] = cfg3_oracle_steps(min(os.cpu_count() or 1, O.openmp_threads()), 10)
    return out


def sweep_at_scale(args, ws, rank):
    """The damping sweep on a large body: BASELINE cfg5's weak-scaling share of one GPU (250 x 250 x 250
    lattice, 15.6 M particles, 1.24 G slots, dp 0.004, 5-layer clamp), where the colours hold ~10^4
    cells and the streamed FAST kernel (slot block from L2) runs; DPU/s against the HBM roofline on the
    same algorithmic byte model as the headline, with the DRAM bytes per launch of the committed ncu
    capture (profiles/traffic_scale.json)."""
    from paper_2103_08932_b200 import scenarios as S
    cfg = S.cfg5_weak()
    d = S.build_device(cfg, prepare=False)
    d.set_reduction("fast")
    offsets = d.row_offsets()
    s_free, n_free = free_slots(offsets, cfg["constrained"])
    b_sweep = 2 * (BYTES_SLOT * s_free + P_D[3] * n_free)
    eta_t, dt = cfg["eta"] / cfg["alpha"], 1e-5
    d.damping_sweep("particle_split", eta_t, dt, count=2)
    sweeps = max(3, min(args.scale_sweeps, 50))
    elapsed = d.damping_sweep("particle_split", eta_t, dt, count=sweeps)
    t_max = barrier_and_max(elapsed, ws)
    t_sweep = t_max / sweeps
    peak, peak_src = load_peaks()
    achieved = b_sweep / t_sweep / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic_scale.json")) as fh:
            traffic = json.load(fh)
    except Exception:
        pass
    del d
    return {"metric": "damping pair-updates/s (fp64 particle-split Strang sweep)",
            "value": 2 * s_free * sweeps * ws / t_max, "unit": "DPU/s", "sweeps": sweeps,
            "ms_per_sweep": t_sweep * 1e3,
            "config": {"workload": "cfg5 weak-scaling share of one GPU: 250^3 lattice dp 0.004, 5-layer clamp",
                       "particles": len(cfg["r0"]), "slots": int(offsets[-1]), "reduction": "fast",
                       "sweep_tiling": "auto (streamed: colours of ~9,700 cells)"},
            "roofline": {"bound": "hbm", "kernel": "k_sweep_fast<streamed> (one colour phase)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "bytes_per_launch": b_sweep / 54, "avg_launch_s": t_sweep / 54,
                         "traffic": traffic, "peak_source": peak_src}}


def sweep_sharded(args, ws, rank):
    """N > 1: BASELINE cfg5's weak-scaling run. A body of ws x `--scale-layers` x-layers of 250 x 250
    (dp 0.004; 15.6 M particles per GPU at the default 250) is x-slab decomposed, one slab per rank,
    with the fused exchange across processes (slabs.IpcSlabSweep: CUDA IPC mappings of the
    neighbours' velocity arrays, phase kernels storing shared columns into them over NVLink, the
    per-phase barrier as stream waits on the neighbours' IPC phase events). Device time per rank
    (events on the slab's stream), max over ranks; DPU over the whole body. Compare with
    `sweep_at_scale` of the N = 1 line for the weak-scaling efficiency of the decomposed sweep."""
    import numpy as np
    import torch.distributed as dist

    from paper_2103_08932_b200 import scenarios as S
    from paper_2103_08932_b200 import slabs

    from paper_2103_08932_b200 import dev

    layers, dp = args.scale_layers, 0.004
    h = 1.3 * dp
    # this rank's held particles only (slabs.lattice_slab == decompose on the whole lattice)
    grid, ranges, part, r0 = slabs.lattice_slab([0.0, 0.0, 0.0], [layers * ws * dp, 1.0, 1.0], dp, h, ws, rank)
    parts = [slabs.Slab(r, x0, x1, None) for r, (x0, x1) in enumerate(ranges)]
    cons_local = (r0[:, 0] < 5 * dp).astype(np.uint8)
    d = dev.DeviceSystem(r0, dp ** 3, S.RHO0, h, cons_local, grid=grid[:2])
    d.set_task_range(part.x0, part.x1)
    cols = slabs.cell_columns(r0, grid[0], grid[2], grid[1][0])
    own = (cols >= part.x0) & (cols < part.x1)
    del r0
    d.set_reduction("fast")
    off = d.row_offsets()
    rows = off[1:] - off[:-1]
    s_free_local = int(rows[own & (cons_local == 0)].sum())
    gloo = dist.new_group(backend="gloo")
    sweep = slabs.IpcSlabSweep(d, rank, ws, group=gloo)
    eta_t, dt = S.eta_for(h), 1e-5
    sweep.sweep("particle_split", eta_t, dt, count=2)
    sweeps = max(3, min(args.scale_sweeps, 50))
    dist.barrier(group=gloo)
    d.timer_start()
    sweep.sweep("particle_split", eta_t, dt, count=sweeps)
    t = d.timer_stop()
    t_max = barrier_and_max(t, ws)
    tot = [None] * ws
    dist.all_gather_object(tot, (s_free_local, int(own.sum())), group=gloo)
    s_free = sum(x[0] for x in tot)
    n_owned = sum(x[1] for x in tot)
    # the full loop over the slabs (cfg5: TL-SPH step + random-choice damping, alpha 0.2): halo
    # pushes and sweeps through the IPC links, dt from an all-reduce of the step scalars
    loop = None
    if args.scale_steps > 0:
        mat = S.material()
        g = np.zeros((d.n, 3))
        g[:, 1] = -S.GRAVITY
        d.set("body", g)
        d.prepare(mat)
        group = slabs.IpcGroup(slabs.DeviceSlabEngine(d, 3), [(p.x0, p.x1) for p in parts], rank, sweep)
        spec = slabs.LoopSpec(mat, h, S.eta_for(h), 0.2, args.scale_steps, seed=0)
        dist.barrier(group=gloo)
        d.timer_start()
        res = slabs.run_loop(group, spec, 3, sweeper=lambda scheme, et, dt_: sweep.sweep(scheme, et, dt_))
        t_loop = barrier_and_max(d.timer_stop(), ws)
        loop = {"metric": "particle-steps/s (fp64 TL-SPH step + splitting damping, random choice)",
                "value": n_owned * res["steps"] / t_loop, "unit": "PS/s", "steps": res["steps"],
                "damped_steps": res["damped"], "ms_per_step": t_loop / res["steps"] * 1e3,
                "exchange": "halo pushes and sweeps through CUDA IPC; dt from an all-reduce per step"}
    sweep.close()
    del d
    peak, peak_src = load_peaks()
    b_sweep = 2 * (BYTES_SLOT * s_free + P_D[3] * n_owned)  # whole body; per GPU divide by ws
    return {"metric": "damping pair-updates/s (fp64 particle-split Strang sweep)",
            "value": 2 * s_free * sweeps / t_max, "unit": "DPU/s", "sweeps": sweeps, "ms_per_sweep": t_max / sweeps * 1e3,
            "scaling": "weak",
            "config": {"workload": f"cfg5 weak scaling: {layers * ws} x 250 x 250 lattice (dp 0.004), "
                                   f"{ws} x-slabs, one per GPU", "particles": n_owned, "slots_free": s_free,
                       "exchange": "fused: CUDA IPC peer stores of shared columns + IPC phase events (no host sync)"},
            "roofline": {"bound": "hbm", "achieved_per_gpu": b_sweep / ws / (t_max / sweeps) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": b_sweep / ws / (t_max / sweeps) / 1e9 / peak,
                         "peak_source": peak_src},
            "timing": "CUDA events on each slab's stream between a barrier and the last phase, max over ranks",
            "loop": loop}


def cfg3_oracle_steps(threads, steps):
    """Reference CPU path (oracle port, OpenMP) over the first `steps` cfg3 loop steps."""
    from oracle import oracle as O
    from paper_2103_08932_b200 import scenarios as S
    cfg = S.cfg3()
    o = O.OracleSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"], constrained=cfg["constrained"])
    o.set_material(S.E_MOD, S.NU, S.RHO0)
    o.set("v", cfg["v0"])
    o.set("body", cfg["body"])
    o.prepare(threads=threads)
    ro = o.run(eta=cfg["eta"], alpha=cfg["alpha"], steps=steps, seed=cfg["seed"], threads=threads)
    n = len(cfg["r0"])
    return {"value": n * ro["steps"] / ro["total_s"], "unit": "PS/s", "cores": threads, "kind": "port",
            "sample": f"first {ro['steps']} cfg3 loop steps, oracle OpenMP"}


def reference_particle_steps():
    from oracle import oracle as O
    threads = min(os.cpu_count() or 1, O.openmp_threads())
    b = cfg3_oracle_steps(threads, 10)
    return {"metric": "particle-steps/s (fp64 TL-SPH step + splitting damping, random choice)",
            "value": b["value"], "unit": "PS/s", "impl": "reference", "cpu_baseline": b}


def run_reference(args, ws, rank):
    """--impl reference: the reference CPU path (oracle port; the reference itself cannot be built here)."""
    if rank != 0:
        return None
    from oracle import oracle as O
    from paper_2103_08932_b200 import scenarios as S
    cfg = S.cfg2()
    threads = min(os.cpu_count() or 1, O.openmp_threads())
    o = O.OracleSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"])
    o.set("v", cfg["v0"])
    nb = o.neighborhood()
    s_free = int(nb["offsets"][-1])
    dpu = 2 * s_free
    eta_t = cfg["eta"] / cfg["alpha"]
    for _ in range(max(0, min(args.warmup, 3))):
        o.damping_sweep("particle_split", eta_t, cfg["fixed_dt"], threads=threads)
    budget = args.cpu_budget * 4
    times = []
    t_start = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        o.damping_sweep("particle_split", eta_t, cfg["fixed_dt"], threads=threads)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget:
            break
    total = sum(times)
    value = dpu * len(times) / total
    return {
        "impl": "reference",
        "metric": "damping pair-updates/s (fp64 particle-split Strang sweep)",
        "value": value, "unit": "DPU/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total / len(times) * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded 64^3 lattice, v ~ N(0,1))",
        "config": {"workload": "cfg2: 3D damping-only sweep, 64^3 lattice, 27-colour particle-split, alpha=1",
                   "particles": len(cfg["r0"]), "slots": s_free},
        "cpu_baseline": {"value": value, "unit": "DPU/s", "cores": threads, "kind": "port",
                         "sample": f"{len(times)} of {args.steps} requested full sweeps (time budget {budget:.0f} s)"},
        "e2e": {"value": value, "unit": "DPU/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=["cfg2"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of CPU sampling")
    ap.add_argument("--ps-steps", type=int, default=300, help="loop steps of the particle-steps/s leg (cfg3)")
    ap.add_argument("--no-ps", action="store_true", help="skip the particle-steps/s leg")
    ap.add_argument("--scale-sweeps", type=int, default=10, help="sweeps of the large-body (cfg5-weak) leg")
    ap.add_argument("--no-scale", action="store_true", help="skip the large-body sweep leg")
    ap.add_argument("--scale-steps", type=int, default=20, help="loop steps of the N > 1 sharded leg (0: sweep only)")
    ap.add_argument("--scale-layers", type=int, default=250,
                    help="x-layers of 250 x 250 per GPU of the N > 1 sharded leg (cfg5 weak scaling)")
    ap.add_argument("--parity-sweeps", type=int, default=500, help="cfg2 sweeps of the GPU-vs-oracle check (0: skip)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)
    ws, rank, local = dist_env()
    # TLSPH_BENCH_ONE_DEVICE=1: every rank on GPU 0 over gloo (protocol tests of the N > 1 path on a
    # one-GPU box; small --scale-layers)
    one_device = os.environ.get("TLSPH_BENCH_ONE_DEVICE") == "1"
    if one_device:
        local = 0
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("gloo" if one_device else "nccl")
    if args.impl == "reference":
        out = run_reference(args, ws, rank)
        if out is not None and not args.no_ps:
            out["particle_steps"] = reference_particle_steps()
    else:
        from paper_2103_08932_b200 import dev
        dev.select_device(local)
        out = run_cfg2(args, ws, rank)
        if not args.no_ps:
            out["particle_steps"] = particle_steps(args, ws, rank)
        if not args.no_scale:
            if ws == 1:
                out["sweep_at_scale"] = sweep_at_scale(args, ws, rank)
            else:
                sh = sweep_sharded(args, ws, rank)
                if out is not None:
                    out["sweep_sharded"] = sh
    if rank == 0 and out is not None:
        print(json.dumps(out))
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
