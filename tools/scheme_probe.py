"""Sweep time per scheme and reduction mode (particle split / pairwise split; fast / ordered):
  python tools/scheme_probe.py [cfg2|cfg3|cfg4|cfg5_weak]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08932_b200 import scenarios as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = getattr(S, name)()
d = S.build_device(cfg, prepare=False)
slots = d.slot_count
eta_t = cfg["eta"] / cfg["alpha"]
for scheme in ("particle_split", "pairwise_split"):
    for mode in ("fast", "ordered"):
        d.set_reduction(mode)
        d.damping_sweep(scheme, eta_t, cfg["fixed_dt"] or 1e-5)
        el = d.damping_sweep(scheme, eta_t, cfg["fixed_dt"] or 1e-5, count=3) / 3
        print(f"{name} {scheme:15s} {mode:8s} {el * 1e3:8.3f} ms/sweep  {2 * slots / el / 1e9:6.1f} G DPU/s", flush=True)
