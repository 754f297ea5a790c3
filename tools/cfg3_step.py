"""cfg3 (640,000-particle beam) device loop, FAST: a few steps, for per-kernel launch lists
(ncu -k regex:'k_stress|k_momentum|k_deformation|k_step_begin')."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08932_b200 import scenarios as S  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = S.cfg3()
d = S.build_device(cfg, prepare=True)
d.set_reduction("fast")
r = d.run(S.material(), eta=cfg["eta"], alpha=cfg["alpha"], steps=steps, seed=cfg["seed"])
print(f"cfg3 n={d.n} slots={d.slot_count} steps={r['steps']} elastic {r['elastic_s'] / r['steps'] * 1e3:.3f} ms/step "
      f"damping {r['damping_s'] * 1e3:.1f} ms ({r['damped']} sweeps)", flush=True)
