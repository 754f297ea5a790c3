"""cfg2 pairwise-split FAST sweep: first call (cold: module load, factor array) vs warm calls."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08932_b200 import scenarios as S  # noqa: E402

cfg = S.cfg2()
d = S.build_device(cfg, prepare=False)
d.set_reduction("fast")
eta_t, dt = cfg["eta"] / cfg["alpha"], cfg["fixed_dt"]
d.damping_sweep("particle_split", eta_t, dt, count=3)
for rep in range(4):
    el = d.damping_sweep("pairwise_split", eta_t, dt, count=5)
    print(f"pairwise call {rep}: {el / 5 * 1e3:.3f} ms per sweep", flush=True)
