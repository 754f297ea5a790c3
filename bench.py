#!/usr/bin/env python3
"""Benchmark of the B200 hot path (BASELINE.json metric), one JSON line on rank 0.

Headline (N = 1): BASELINE configs[3] (cfg4), the largest configuration that fits one GPU --
a jittered 1 x 1 x 0.5 m block at dp 0.004 (7,812,500 particles, ~560 M neighbour slots), fp64
TL-SPH step + random-choice splitting damping (alpha 0.1), stable_dt, per-step current-cell
rebuild. One step = one iteration of runner.cpp:341-391 over the whole body.
metric = particle-steps per second (PS/s). The timed window is loop steps W .. W+K-1 (after W
untimed warm-up steps of the same run); the reference arm times the same window.

  python bench.py [--gpus N] [--steps K] [--warmup W]
  python bench.py --impl reference ...   # the reference CPU path (oracle port, all host cores)

Keys of the line:
  value      PS/s from CUDA events on the library's stream around the K steps (inputs resident);
  e2e        the same metric through the reference's C++ operator API (stable_dt / verlet_step /
             strang_damping_sweep<3> on a host ParticleSystem<3> whose storage the caller page-locks
             once (tlsph::pin_host_memory); every call moves the fields the reference operator reads
             host -> device and the ones it writes device -> host; lib/tlsph-operator-loop);
  roofline   the TL-SPH step kernels (k_step_begin + passes A-C + current-cell rebuild) against
             the measured HBM copy bandwidth on BASELINE.md §4's algorithmic byte model;
  cpu_baseline / parity   the oracle (reference arithmetic, OpenMP on every host core) over the
             same W+K steps; its K timed steps are the baseline, its final state the parity check;
  legs       cfg2 damping sweep (DPU/s, its e2e through strang_damping_sweep<3>, 500-sweep parity),
             pairwise split sweep on cfg2, cfg1 full run, cfg3 loop, cfg5 weak-scaling share
             (sweep DPU/s and loop PS/s on one GPU: the N = 1 base of the N > 1 line), and the
             paper's Table 1 damping times (bending cantilever h/dp 12, t = 2 s) through tlsph_sim_run.

Multi-GPU (torchrun, one rank per GPU): value = BASELINE cfg5's weak-scaling loop, one x-slab of
an N x 250-layer body (15.6 M particles) per rank, driven through the C entry point
tlsph_dev_group_run (csrc/cuda/group.cu: CUDA IPC peer stores per colour phase and halo pushes,
dt all-reduce over a gloo communicator), PS/s over the whole body, device time max over ranks.
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
OPERATOR_LOOP = os.path.join(ROOT, "paper_2103_08932_b200", "lib", "tlsph-operator-loop")

METRIC_PS = "particle-steps/s (fp64 TL-SPH step + random-choice splitting damping)"
METRIC_DPU = "damping pair-updates/s (fp64 particle-split Strang sweep)"


# ----------------------------------------------------------------------------- plumbing
def load_json(rel):
    try:
        with open(os.path.join(ROOT, rel)) as fh:
            return json.load(fh)
    except Exception:
        return None


def load_peaks():
    pk = load_json("MEASURED_PEAKS.json")
    if pk and "hbm_gbs" in pk:
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
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
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), \
        int(os.environ.get("LOCAL_RANK", "0"))


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


def cpu_threads():
    from oracle import oracle as O  # the checker / CPU baseline only
    return min(os.cpu_count() or 1, O.openmp_threads())


def rel_l2(a, b):
    import numpy as np
    a, b = np.asarray(a, dtype=np.float64).ravel(), np.asarray(b, dtype=np.float64).ravel()
    den = float(np.linalg.norm(b))
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def free_slots(off, cons):
    if cons is None:
        return int(off[-1]), len(off) - 1
    counts = off[1:] - off[:-1]
    free = cons == 0
    return int(counts[free].sum()), int(free.sum())


def step_bytes(n, slots):
    """algorithmic bytes of one elastic step (3D): S*2*(4+8+24) + N*P_s."""
    return slots * 2 * (4 + 8 + 8 * 3) + n * P_S[3]


def sweep_bytes(s_free, n_free, dim=3):
    return 2 * (BYTES_SLOT * s_free + P_D[dim] * n_free)


def operator_loop(what, steps, warmup):
    """The e2e legs: lib/tlsph-operator-loop (C++ against include/tlsph/*.hpp only)."""
    out = subprocess.run([OPERATOR_LOOP, what, str(steps), str(warmup), "fast"], capture_output=True, text=True,
                         timeout=1200)
    if out.returncode != 0:
        raise RuntimeError(f"tlsph-operator-loop {what} failed: {out.stderr.strip()[-400:]}")
    return json.loads(out.stdout.strip().splitlines()[-1])


# ----------------------------------------------------------------------------- shared config (both arms)
CFG4_WORKLOAD = ("cfg4: jittered 1 x 1 x 0.5 m block, dp 0.004 (250 x 250 x 125 lattice, +-0.4 dp jitter "
                 "from RandomSource(3)), fp64 neo-Hookean TL-SPH + random-choice particle-split damping "
                 "(alpha 0.1, seed 0), gravity, 5-layer clamp, stable_dt (CFL 0.6)")


def cfg4_config(n, slots, steps, warmup):
    return {"workload": CFG4_WORKLOAD, "particles": int(n), "slots": int(slots),
            "window": f"loop steps {warmup}..{warmup + steps - 1} of one run (after {warmup} warm-up steps)",
            "l2": "inputs larger than L2 (neighbour CSR ~30 GB, state ~3 GB vs 126 MB L2); no flush"}


# ----------------------------------------------------------------------------- headline, ours (N = 1)
def headline_cfg4(args):
    import numpy as np

    from paper_2103_08932_b200 import scenarios as S
    cfg = S.cfg4()
    mat = S.material()
    d = S.build_device(cfg, prepare=True)
    d.set_reduction("fast")
    d.set_resort(True)
    n, slots = int(d.n), int(d.slot_count)
    W, K = args.warmup, args.steps
    kw = dict(eta=cfg["eta"], alpha=cfg["alpha"], seed=cfg["seed"])
    w = d.run(mat, steps=W, **kw) if W > 0 else None
    cuda_sync()
    with ClockSampler(0) as clk:
        r = d.run(mat, steps=W + K, resume=W > 0, **kw)
    cuda_sync()
    base = w or {"total_s": 0.0, "elastic_s": 0.0, "damping_s": 0.0, "damped": 0}  # times are cumulative
    t = r["total_s"] - base["total_s"]
    t_el = (r["elastic_s"] - base["elastic_s"]) / K
    damped = r["damped"] - base["damped"]
    t_dm = (r["damping_s"] - base["damping_s"]) / max(damped, 1)
    assert r["steps"] == W + K
    final = {"v": d.get("v"), "u": d.get("r") - cfg["r0"], "steps": r["steps"], "damped": r["damped"], "t": r["t"]}
    peak, peak_src = load_peaks()
    b_el = step_bytes(n, slots)
    off = d.row_offsets()
    s_free, n_free = free_slots(off, cfg["constrained"])
    b_sw = sweep_bytes(s_free, n_free)
    traffic = load_json("profiles/traffic_cfg4.json")
    out = {
        "metric": METRIC_PS,
        "value": n * K / t, "unit": "PS/s", "n_gpus": 1, "steps": K, "warmup": W,
        "ms_per_step": t / K * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded jittered lattice, BASELINE.md §3)",
        "config": cfg4_config(n, slots, K, W),
        "mode": {"reduction": "fast (lane-parallel sums; <= 1e-10 of the reference order)",
                 "resort": ("per-step current-position cell binning (keys, counting sort, in-cell order) inside "
                            "the loop's graph, its time included; not a storage permutation: the CSR, colouring "
                            "and sweep order are r0-based (SURVEY.md §7 item 7), storage keeps r0-cell order")},
        "damped_steps": damped, "elastic_ms_per_step": t_el * 1e3, "damping_ms_per_damped_step": t_dm * 1e3,
        "roofline": {"bound": "hbm", "kernel": "TL-SPH step: k_step_begin + passes A, B, C (+ current-cell binning)",
                     "achieved": b_el / t_el / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": b_el / t_el / 1e9 / peak, "bytes_per_launch": b_el, "avg_launch_s": t_el,
                     "traffic": traffic.get("dram_bytes_per_step") if traffic else None,
                     "traffic_source": traffic.get("source") if traffic else None, "peak_source": peak_src,
                     "timing": "CUDA events on the library's stream around each step's kernels, timed steps only"},
        "roofline_damping": {"bound": "hbm", "kernel": "k_sweep_folds + 54 colour phases (k_sweep_fast, streamed)",
                             "achieved": b_sw / t_dm / 1e9, "peak": peak, "unit": "GB/s",
                             "frac": b_sw / t_dm / 1e9 / peak, "bytes_per_sweep": b_sw},
        "gpu_launches": r["kernel_launches"],  # this call's launches (the timed K steps)
        "clocks": clk.summary(),
    }
    del d
    return out, cfg, final


def oracle_loop(cfg, W, K, threads):
    """The reference CPU path (oracle port of runner.cpp:341-391) on a scenario: W warm-up steps,
    then K timed steps of the same run."""
    from oracle import oracle as O
    from paper_2103_08932_b200 import scenarios as S
    t0 = time.perf_counter()
    o = O.OracleSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"], constrained=cfg["constrained"])
    o.set_material(S.E_MOD, S.NU, S.RHO0)
    o.set("v", cfg["v0"])
    o.set("body", cfg["body"])
    o.prepare(threads=threads)
    init_s = time.perf_counter() - t0
    kw = dict(eta=cfg["eta"], alpha=cfg["alpha"], seed=cfg["seed"], threads=threads)
    if W > 0:
        o.run(steps=W, **kw)
    r = o.run(steps=W + K, resume=W > 0, **kw)
    return o, r, init_s


# ----------------------------------------------------------------------------- legs (N = 1)
def leg_cfg2(args):
    """cfg2: 64^3 damping-only sweep, DPU/s; e2e through tlsph::strang_damping_sweep<3>; parity."""
    import numpy as np

    from paper_2103_08932_b200 import scenarios as S
    cfg = S.cfg2()
    d = S.build_device(cfg, prepare=False)
    d.set_reduction("fast")
    off = d.row_offsets()
    s_free, n_free = free_slots(off, cfg["constrained"])
    eta_t, dt = cfg["eta"] / cfg["alpha"], cfg["fixed_dt"]
    sweeps = max(20, args.steps)
    d.damping_sweep("particle_split", eta_t, dt, count=3)
    el = d.damping_sweep("particle_split", eta_t, dt, count=sweeps)
    peak, _ = load_peaks()
    b = sweep_bytes(s_free, n_free)
    out = {"metric": METRIC_DPU, "value": 2 * s_free * sweeps / el, "unit": "DPU/s", "sweeps": sweeps,
           "ms_per_sweep": el / sweeps * 1e3,
           "config": {"workload": "cfg2: 64^3 lattice, v ~ N(0,1) (seed 1), particle-split, alpha 1, dt 0.6 h / c",
                      "particles": int(d.n), "slots": int(off[-1])},
           "roofline": {"bound": "hbm", "kernel": "k_sweep_fast (staged) x 54 + k_sweep_folds",
                        "achieved": b / (el / sweeps) / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": b / (el / sweeps) / 1e9 / peak, "bytes_per_sweep": b,
                        "traffic": (load_json("profiles/traffic.json") or {}).get("dram_bytes_per_launch"),
                        "note": "latency-bound by construction: 27-particle Gauss-Seidel chains, ~580 cells per colour"}}
    d.damping_sweep("pairwise_split", eta_t, dt, count=1)  # warm-up: kernel load, the per-(eta, dt) factor array
    pw = d.damping_sweep("pairwise_split", eta_t, dt, count=max(5, sweeps // 4))
    npw = max(5, sweeps // 4)
    out["pairwise_split"] = {"value": 2 * s_free * npw / pw, "unit": "DPU/s", "ms_per_sweep": pw / npw * 1e3,
                             "roofline_frac": b / (pw / npw) / 1e9 / peak,
                             "kernel": "k_pair_factors + k_sweep_pairwise (FAST: affine warp scans)"}
    if args.parity_sweeps > 0 and not args.no_cpu:
        from oracle import oracle as O
        threads = cpu_threads()
        d.set("v", cfg["v0"])
        d.damping_sweep("particle_split", eta_t, dt, count=args.parity_sweeps)
        vg = d.get("v")
        o = O.OracleSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"], constrained=cfg["constrained"])
        o.set("v", cfg["v0"])
        times = []
        for _ in range(args.parity_sweeps):
            t0 = time.perf_counter()
            o.damping_sweep("particle_split", eta_t, dt, threads=threads)
            times.append(time.perf_counter() - t0)
        vo = o.get("v")
        out["parity"] = {"sweeps": args.parity_sweeps, "var_v0": float(np.var(cfg["v0"])),
                         "var_gpu": float(np.var(vg)), "var_oracle": float(np.var(vo)),
                         "rel_l2_v": rel_l2(vg, vo), "tolerance": 1e-10, "mode": "fast vs oracle"}
        out["cpu_baseline"] = {"value": 2 * s_free / statistics.median(times), "unit": "DPU/s", "cores": threads,
                               "kind": "port", "sample": f"{len(times)} full cfg2 sweeps (median)"}
    del d
    try:
        e = operator_loop("sweep", max(50, args.steps), 3)
        out["e2e"] = {"value": e["value"], "unit": "DPU/s", "h2d_bytes_per_step": e["h2d_bytes_per_step"],
                      "d2h_bytes_per_step": e["d2h_bytes_per_step"], "path": e["api"], "steps": e["steps"],
                      "host_memory": e.get("host_memory")}
    except Exception as exc:  # reported, never silently replaced
        out["e2e"] = {"error": str(exc)}
    return out


def leg_cfg1(args):
    """cfg1 in full: 2D plate, 16,000 particles, 2,000 steps (latency-bound; reported, not the headline)."""
    from paper_2103_08932_b200 import scenarios as S
    cfg = S.cfg1()
    d = S.build_device(cfg, prepare=True)
    d.set_reduction("fast")
    r = d.run(S.material(), eta=cfg["eta"], alpha=cfg["alpha"], steps=cfg["steps"], seed=cfg["seed"])
    n = int(d.n)
    return {"metric": METRIC_PS, "value": n * r["steps"] / r["total_s"], "unit": "PS/s", "steps": r["steps"],
            "damped_steps": r["damped"], "ms_total": r["total_s"] * 1e3,
            "config": {"workload": "cfg1: 2D plate 400 x 40, neo-Hookean, gravity, 4-column clamp, alpha 0.2",
                       "particles": n, "slots": int(d.slot_count)}}


def leg_cfg3(args):
    """cfg3: 3D beam (640,000 particles), 300 loop steps; CPU sample of the same loop."""
    from paper_2103_08932_b200 import scenarios as S
    cfg = S.cfg3()
    d = S.build_device(cfg, prepare=True)
    d.set_reduction("fast")
    steps = 300
    r = d.run(S.material(), eta=cfg["eta"], alpha=cfg["alpha"], steps=steps, seed=cfg["seed"])
    n, slots = int(d.n), int(d.slot_count)
    t_el = r["elastic_s"] / r["steps"]
    peak, _ = load_peaks()
    out = {"metric": METRIC_PS, "value": n * r["steps"] / r["total_s"], "unit": "PS/s", "steps": r["steps"],
           "damped_steps": r["damped"], "ms_per_step": r["total_s"] / r["steps"] * 1e3,
           "elastic_ms_per_step": t_el * 1e3, "damping_ms_per_damped_step": r["damping_s"] / max(r["damped"], 1) * 1e3,
           "config": {"workload": "cfg3: 3D cantilever beam 400 x 40 x 40, neo-Hookean, gravity, 5-layer clamp, "
                                  "alpha 0.2", "particles": n, "slots": slots},
           "roofline": {"bound": "hbm", "kernel": "TL-SPH step: k_step_begin + passes A, B, C",
                        "achieved": step_bytes(n, slots) / t_el / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": step_bytes(n, slots) / t_el / 1e9 / peak}}
    del d
    if not args.no_cpu:
        threads = cpu_threads()
        o, ro, _ = oracle_loop(cfg, 0, 10, threads)
        out["cpu_baseline"] = {"value": n * ro["steps"] / ro["total_s"], "unit": "PS/s", "cores": threads,
                               "kind": "port", "sample": "first 10 cfg3 loop steps"}
    return out


def leg_cfg5_weak(args):
    """cfg5's weak-scaling share of one GPU (250^3 lattice, 15.6 M particles, 1.24 G slots): the
    damping sweep (DPU/s) and the full loop (PS/s, alpha 0.2) -- the N = 1 base of the N > 1 line."""
    from paper_2103_08932_b200 import scenarios as S
    cfg = S.cfg5_weak()
    d = S.build_device(cfg, prepare=True)
    d.set_reduction("fast")
    off = d.row_offsets()
    s_free, n_free = free_slots(off, cfg["constrained"])
    n, slots = int(d.n), int(off[-1])
    peak, _ = load_peaks()
    eta_t, dt = cfg["eta"] / cfg["alpha"], 1e-5
    d.damping_sweep("particle_split", eta_t, dt, count=2)
    sweeps = max(3, min(args.scale_sweeps, 50))
    el = d.damping_sweep("particle_split", eta_t, dt, count=sweeps)
    b = sweep_bytes(s_free, n_free)
    out = {"sweep": {"metric": METRIC_DPU, "value": 2 * s_free * sweeps / el, "unit": "DPU/s", "sweeps": sweeps,
                     "ms_per_sweep": el / sweeps * 1e3,
                     "roofline": {"bound": "hbm", "kernel": "k_sweep_fast (streamed) x 54 + k_sweep_folds",
                                  "achieved": b / (el / sweeps) / 1e9, "peak": peak, "unit": "GB/s",
                                  "frac": b / (el / sweeps) / 1e9 / peak, "bytes_per_sweep": b,
                                  "traffic": load_json("profiles/traffic_scale.json")}},
           "config": {"workload": "cfg5 weak-scaling share of one GPU: 250^3 lattice dp 0.004, 5-layer clamp, "
                                  "gravity, alpha 0.2", "particles": n, "slots": slots}}
    d.set("v", cfg["v0"])
    steps = max(5, args.scale_steps)
    r = d.run(S.material(), eta=cfg["eta"], alpha=cfg["alpha"], steps=steps, seed=cfg["seed"])
    t_el = r["elastic_s"] / r["steps"]
    out["loop"] = {"metric": METRIC_PS, "value": n * r["steps"] / r["total_s"], "unit": "PS/s", "steps": r["steps"],
                   "damped_steps": r["damped"], "ms_per_step": r["total_s"] / r["steps"] * 1e3,
                   "roofline": {"bound": "hbm", "kernel": "TL-SPH step: k_step_begin + passes A, B, C",
                                "achieved": step_bytes(n, slots) / t_el / 1e9, "peak": peak, "unit": "GB/s",
                                "frac": step_bytes(n, slots) / t_el / 1e9 / peak}}
    del d
    return out


PAPER_TABLE1 = {1.0: {"serial_s": 32.82, "parallel_6core_s": 11.61}, 0.2: {"serial_s": 6.66, "parallel_6core_s": 2.38}}


def leg_paper_table1(args):
    """The paper's Table 1 workload: the damping time of the
    bending cantilever at h/dp = 12 to t = 2 s, particle split, alpha 1.0 and 0.2, through
    tlsph_sim_run (the reference's built-in case: 33 x 12 x 12 = 4,752 particles, its 0.04 x 0.016 m
    geometry, cases.cpp:81-82; the paper's runs used 0.1 x 0.04 m on a Ryzen 5 3600). A small body:
    ~11 cells per colour phase, so the sweep is bound by the per-particle Gauss-Seidel chain latency."""
    import ctypes as C

    L = C.CDLL(os.path.join(ROOT, "paper_2103_08932_b200", "lib", "libtlsph.so.1"))
    L.tlsph_sim_create.argtypes = [C.c_char_p, C.POINTER(C.c_char_p), C.c_size_t, C.POINTER(C.c_void_p)]
    L.tlsph_sim_run.argtypes = [C.c_void_p]
    L.tlsph_sim_destroy.argtypes = [C.c_void_p]
    L.tlsph_sim_phase_seconds.argtypes = [C.c_void_p, C.c_char_p]
    L.tlsph_sim_phase_seconds.restype = C.c_double
    L.tlsph_sim_step_count.argtypes = [C.c_void_p]
    L.tlsph_sim_step_count.restype = C.c_uint64
    L.tlsph_sim_damped_step_count.argtypes = [C.c_void_p]
    L.tlsph_sim_damped_step_count.restype = C.c_uint64
    out = {"workload": "bending_cantilever, resolution 12, end_time 2 s, particle split, gpu.reduction fast",
           "metric": "damping process seconds (tlsph_sim_phase_seconds 'damping')", "runs": []}
    for alpha in (1.0, 0.2):
        ov = ["case=bending_cantilever", "resolution=12", "end_time=2.0", f"damping.alpha={alpha}", "output.dir=",
              "gpu.reduction=fast"]
        arr = (C.c_char_p * len(ov))(*[o.encode() for o in ov])
        h = C.c_void_p()
        if L.tlsph_sim_create(None, arr, len(ov), C.byref(h)) != 0 or L.tlsph_sim_run(h) != 0:
            raise RuntimeError("tlsph_sim_run failed")
        rec = {"alpha": alpha, "damping_s": L.tlsph_sim_phase_seconds(h, b"damping"),
               "elastic_s": L.tlsph_sim_phase_seconds(h, b"elastic"), "total_s": L.tlsph_sim_phase_seconds(h, b"total"),
               "steps": int(L.tlsph_sim_step_count(h)), "damped_steps": int(L.tlsph_sim_damped_step_count(h)),
               "paper": PAPER_TABLE1[alpha]}
        rec["paper_parallel_over_ours"] = PAPER_TABLE1[alpha]["parallel_6core_s"] / rec["damping_s"]
        L.tlsph_sim_destroy(h)
        out["runs"].append(rec)
    return out


# ----------------------------------------------------------------------------- N > 1
def sharded_cfg5(args, ws, rank):
    """BASELINE cfg5's weak scaling: a body of ws x `--scale-layers` x-layers of 250 x 250 (dp 0.004;
    15.6 M particles per GPU at 250), x-slab decomposed, one slab per rank, fused cross-process
    exchange (CUDA IPC peer stores + IPC events); loop PS/s and sweep DPU/s over the whole body,
    device time per rank (events on the slab's stream), max over ranks."""
    import numpy as np
    import torch.distributed as dist

    from paper_2103_08932_b200 import dev
    from paper_2103_08932_b200 import scenarios as S
    from paper_2103_08932_b200 import slabs

    layers, dp = args.scale_layers, 0.004
    h = 1.3 * dp
    grid, ranges, part, r0 = slabs.lattice_slab([0.0, 0.0, 0.0], [layers * ws * dp, 1.0, 1.0], dp, h, ws, rank)
    cons = (r0[:, 0] < 5 * dp).astype(np.uint8)
    d = dev.DeviceSystem(r0, dp ** 3, S.RHO0, h, cons, grid=grid[:2])
    d.set_task_range(part.x0, part.x1)
    cols = slabs.cell_columns(r0, grid[0], grid[2], grid[1][0])
    own = (cols >= part.x0) & (cols < part.x1)
    d.set_reduction("fast")
    off = d.row_offsets()
    rows = off[1:] - off[:-1]
    s_free_local = int(rows[own & (cons == 0)].sum())
    slots_local = int(rows[own].sum())
    gloo = dist.new_group(backend="gloo")
    mat = S.material()
    g = np.zeros((d.n, 3))
    g[:, 1] = -S.GRAVITY
    d.set("body", g)
    d.prepare(mat)
    # the C entry point: tlsph_dev_group_* (csrc/cuda/group.cu) over a gloo communicator
    group = slabs.CGroup(d, slabs.TorchComm(gloo))
    W, K = args.warmup, args.steps
    kw = dict(h=h, eta=S.eta_for(h), alpha=0.2, seed=0)
    if W > 0:
        group.run(mat, steps=W, **kw)
    dist.barrier(group=gloo)
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        res = group.run(mat, steps=K, **kw)
        t_loop = barrier_and_max(res["device_s"], ws)
    tot = [None] * ws
    dist.all_gather_object(tot, (s_free_local, int(own.sum()), slots_local), group=gloo)
    n_owned = sum(x[1] for x in tot)
    slots = sum(x[2] for x in tot)
    eta_t, dt = S.eta_for(h) / 0.2, 1e-5
    nsw = max(3, min(args.scale_sweeps, 50))
    dist.barrier(group=gloo)
    d.timer_start()
    group.sweep("particle_split", eta_t, dt, count=nsw)
    t_sw = barrier_and_max(d.timer_stop(), ws)
    group.close()
    peak, peak_src = load_peaks()
    s_free = sum(x[0] for x in tot)
    b_step = step_bytes(n_owned, slots) / ws
    return {"metric": METRIC_PS, "value": n_owned * res["steps"] / t_loop, "unit": "PS/s", "n_gpus": ws,
            "steps": K, "warmup": W, "ms_per_step": t_loop / K * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded lattice, BASELINE.md §3)",
            "config": {"workload": f"cfg5 weak scaling: {layers * ws} x 250 x 250 lattice (dp 0.004), {ws} x-slabs, "
                                   "one per GPU, alpha 0.2", "particles": n_owned, "slots": slots,
                       "parallelism": f"x-slabs x{ws}",
                       "exchange": "fused: CUDA IPC peer stores of shared columns + IPC phase events",
                       "driver": "C ABI tlsph_dev_group_run / tlsph_dev_group_sweep (csrc/cuda/group.cu)"},
            "roofline": {"bound": "hbm", "kernel": "whole step per GPU (elastic + damping share)",
                         "achieved": b_step / (t_loop / K) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": b_step / (t_loop / K) / 1e9 / peak, "peak_source": peak_src},
            "damped_steps": res["damped"],
            "sweep": {"metric": METRIC_DPU, "value": 2 * s_free * nsw / t_sw, "unit": "DPU/s",
                      "ms_per_sweep": t_sw / nsw * 1e3},
            "gpu_launches": res["kernel_launches"],  # rank 0's kernels over the timed K steps (lower bound)
            "e2e": {"value": None, "unit": "PS/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                    "note": "the reference's operator API is a one-process, one-body interface (no slab form): "
                            "its end-to-end figure is the N = 1 line's e2e"},
            "clocks": clk.summary(),
            "timing": "CUDA events on each slab's stream between a barrier and the last step, max over ranks"}


# ----------------------------------------------------------------------------- reference arm
def reference_cfg4_inputs():
    """cfg4's inputs built with the oracle's own lattice and RandomSource (no product library)."""
    import numpy as np
    from oracle import oracle as O
    dp = 0.004
    r0 = O.box_lattice([0.0, 0.0, 0.0], [1.0, 1.0, 0.5], dp)
    n = len(r0)
    u = O.random_uniforms(3, n * 6)
    r0 = np.ascontiguousarray(r0 + (2.0 * u[: n * 3].reshape(n, 3) - 1.0) * (0.4 * dp))
    v0 = -0.01 + 0.02 * u[n * 3:].reshape(n, 3)
    mat = O.material(2.0e6, 0.3, 1000.0)
    h = 1.3 * dp
    body = np.tile([0.0, -9.81, 0.0], (n, 1))
    return dict(r0=r0, V0=dp ** 3, rho0=1000.0, h=h, constrained=(r0[:, 0] < 5 * dp).astype(np.uint8), v0=v0,
                body=body, eta=0.2 * 1000.0 * mat["c"] * h, alpha=0.1, seed=0)


def run_reference(args, ws, rank):
    """--impl reference: the reference CPU path (oracle port of runner.cpp:341-391 and the operators it
    calls; the reference itself cannot be built here) on every host core, same config and window."""
    if rank != 0:
        return None
    from oracle import oracle as O
    threads = cpu_threads()
    cfg = reference_cfg4_inputs()
    W, K = args.warmup, args.steps
    t0 = time.perf_counter()
    o = O.OracleSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"], constrained=cfg["constrained"])
    o.set_material(2.0e6, 0.3, 1000.0)
    o.set("v", cfg["v0"])
    o.set("body", cfg["body"])
    o.prepare(threads=threads)
    init_s = time.perf_counter() - t0
    n = len(cfg["r0"])
    slots = int(o.neighborhood([])["offsets"][-1])
    kw = dict(eta=cfg["eta"], alpha=cfg["alpha"], seed=cfg["seed"], threads=threads)
    if W > 0:
        o.run(steps=W, **kw)
    r = o.run(steps=W + K, resume=W > 0, **kw)
    value = n * K / r["total_s"]
    return {
        "impl": "reference", "metric": METRIC_PS, "value": value, "unit": "PS/s", "n_gpus": ws, "steps": K,
        "warmup": W, "ms_per_step": r["total_s"] / K * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded jittered lattice, BASELINE.md §3)",
        "config": cfg4_config(n, slots, K, W),
        "cpu_baseline": {"value": value, "unit": "PS/s", "cores": threads, "kind": "port",
                         "sample": f"cfg4 loop steps {W}..{W + K - 1} (oracle restatement of runner.cpp:341-391, "
                                   f"OpenMP on {threads} threads); init {init_s:.1f} s untimed"},
        "e2e": {"value": value, "unit": "PS/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "damped_steps": int(r["damped"]),
    }


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle legs (cpu_baseline, parity)")
    ap.add_argument("--no-legs", action="store_true", help="headline only")
    ap.add_argument("--no-e2e", action="store_true", help="skip the operator-API e2e leg of the headline")
    ap.add_argument("--parity-sweeps", type=int, default=500, help="cfg2 sweeps of the GPU-vs-oracle check")
    ap.add_argument("--scale-sweeps", type=int, default=10, help="sweeps of the cfg5-weak legs")
    ap.add_argument("--scale-steps", type=int, default=20, help="loop steps of the cfg5-weak leg (N = 1)")
    ap.add_argument("--scale-layers", type=int, default=250, help="x-layers of 250 x 250 per GPU (N > 1)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)
    args.steps = max(args.steps, 1)
    ws, rank, local = dist_env()
    one_device = os.environ.get("TLSPH_BENCH_ONE_DEVICE") == "1"  # N > 1 protocol on one GPU (tests)
    if one_device:
        local = 0
    if ws > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "ours":
            torch.cuda.set_device(local)
        dist.init_process_group("gloo" if (one_device or args.impl == "reference") else "nccl")
    if args.impl == "reference":
        out = run_reference(args, ws, rank)
    else:
        from paper_2103_08932_b200 import dev
        dev.select_device(local)
        if ws > 1:
            out = sharded_cfg5(args, ws, rank)
        else:
            out, cfg, final = headline_cfg4(args)
            if not args.no_e2e:
                try:
                    e = operator_loop("loop", args.steps, args.warmup)
                    out["e2e"] = {"value": e["value"], "unit": "PS/s", "h2d_bytes_per_step": e["h2d_bytes_per_step"],
                                  "d2h_bytes_per_step": e["d2h_bytes_per_step"], "path": e["api"],
                                  "host_memory": e.get("host_memory"),
                                  "ms_per_step": e["seconds"] / max(args.steps, 1) * 1e3,
                                  "caller_host_ms_per_step": (e.get("caller_host_seconds", 0.0) /
                                                              max(args.steps, 1) * 1e3),
                                  "caller_host_note": "the reference runner's own serial host code inside the "
                                                      "timed loop (check_finite, runner.cpp:233-247; "
                                                      "apply_constraints), not part of the operator API",
                                  "window": f"steps {args.warmup}..{args.warmup + args.steps - 1}",
                                  "damped_steps": e["damped_steps"]}
                except Exception as exc:
                    out["e2e"] = {"error": str(exc)}
            if not args.no_cpu:
                threads = cpu_threads()
                o, ro, init_s = oracle_loop(cfg, args.warmup, args.steps, threads)
                out["cpu_baseline"] = {"value": len(cfg["r0"]) * args.steps / ro["total_s"], "unit": "PS/s",
                                       "cores": threads, "kind": "port",
                                       "sample": f"cfg4 loop steps {args.warmup}..{args.warmup + args.steps - 1}, "
                                                 f"oracle OpenMP on {threads} threads (init {init_s:.1f} s untimed)"}
                out["parity"] = {"steps": int(ro["steps"]), "steps_gpu": int(final["steps"]),
                                 "damped_oracle": int(ro["damped"]), "damped_gpu": int(final["damped"]),
                                 "t_rel_diff": abs(final["t"] - ro["t"]) / ro["t"],
                                 "rel_l2_v": rel_l2(final["v"], o.get("v")),
                                 "rel_l2_displacement": rel_l2(final["u"], o.get("r") - cfg["r0"]),
                                 "tolerance": 1e-10, "mode": "fast + re-sort (GPU) vs oracle, same W+K steps"}
                del o
            if not args.no_legs:
                for name, fn in (("sweep_cfg2", leg_cfg2), ("cfg1", leg_cfg1), ("particle_steps_cfg3", leg_cfg3),
                                 ("cfg5_weak", leg_cfg5_weak), ("paper_table1", leg_paper_table1)):
                    try:
                        out[name] = fn(args)
                    except Exception as exc:
                        out[name] = {"error": f"{type(exc).__name__}: {exc}"}
    if rank == 0 and out is not None:
        print(json.dumps(out))
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
