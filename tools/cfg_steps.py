"""K device-loop steps (FAST, per-step current-cell rebuild) of a BASELINE scenario, for ncu captures
and launch lists:  python tools/cfg_steps.py cfg4 [--steps K] [--sweeps M] [--resort]

Builds the scenario on the device (prepare = runner.cpp:306-312), runs M standalone damping sweeps
and K loop steps (runner.cpp:341-391), prints per-step elastic / damping times from the loop's events.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08932_b200 import scenarios as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="cfg4")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--sweeps", type=int, default=1)
ap.add_argument("--resort", action="store_true")
ap.add_argument("--mode", default="fast")
a = ap.parse_args()
cfg = getattr(S, a.config)()
d = S.build_device(cfg, prepare=True)
d.set_reduction(a.mode)
if a.resort:
    d.set_resort(True)
eta_t = cfg["eta"] / cfg["alpha"]
if a.sweeps:
    el = d.damping_sweep("particle_split", eta_t, cfg["fixed_dt"] or 1e-5, count=a.sweeps)
    print(f"{a.config}: {a.sweeps} sweeps {el / a.sweeps * 1e3:.3f} ms per sweep", flush=True)
if a.steps:
    r = d.run(S.material(), eta=cfg["eta"], alpha=cfg["alpha"], steps=a.steps, seed=cfg["seed"])
    print(f"{a.config}: n={d.n} slots={d.slot_count} steps={r['steps']} damped={r['damped']} "
          f"elastic {r['elastic_s'] / r['steps'] * 1e3:.3f} ms/step, damping {r['damping_s'] * 1e3:.3f} ms total, "
          f"{d.n * r['steps'] / r['total_s'] / 1e9:.3f} G PS/s", flush=True)
