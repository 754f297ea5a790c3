"""Sweep throughput across body sizes (FAST particle split): cfg2, cfg3, cfg4, cfg5-weak.

  python tools/sweep_sizes.py [cfg2 cfg3 cfg4 cfg5_weak] [--sweeps K]

Per body: 2 untimed sweeps, then K sweeps timed on the library's stream (tlsph_dev_damping_sweeps),
printed as ms per sweep and G DPU/s (2 x free slots per sweep). The slot-block
mode of the sweep kernel follows TLSPH_SWEEP_STREAM (unset: automatic).
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08932_b200 import scenarios as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", default=["cfg2", "cfg3", "cfg4", "cfg5_weak"])
ap.add_argument("--sweeps", type=int, default=10)
a = ap.parse_args()
mode = os.environ.get("TLSPH_SWEEP_STREAM", "auto")
for name in a.configs:
    cfg = getattr(S, name)()
    d = S.build_device(cfg, prepare=False)
    d.set_reduction("fast")
    eta = cfg["eta"] / cfg["alpha"]
    dt = cfg["fixed_dt"] or 1e-5
    d.damping_sweep("particle_split", eta, dt, count=2)
    el = d.damping_sweep("particle_split", eta, dt, count=a.sweeps) / a.sweeps
    dpu = 2 * d.slot_count  # clamped rows (cfg3-5: 1-2 %) included
    print(f"{name} stream={mode}: n={d.n} slots={d.slot_count} sweep {el * 1e3:.3f} ms = "
          f"{dpu / el / 1e9:.1f} G DPU/s", flush=True)
    del d
