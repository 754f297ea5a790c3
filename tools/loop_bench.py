"""Particle-steps/s of the device-resident TL-SPH + splitting-damping loop (runner.cpp:341-391) on
BASELINE configs 1 and 3: fixed step counts, elastic vs damping time from the loop's own events."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08932_b200 import scenarios as S  # noqa: E402

for name, steps in (("cfg1", 2000), ("cfg3", 300)):
    cfg = getattr(S, name)()
    t0 = time.perf_counter()
    d = S.build_device(cfg, prepare=True)
    t_init = time.perf_counter() - t0
    for mode in ("fast", "ordered"):
        d2 = S.build_device(cfg, prepare=True)
        d2.set_reduction(mode)
        r = d2.run(S.material(), eta=cfg["eta"], alpha=cfg["alpha"], steps=steps, seed=cfg["seed"])
        ps = d2.n * r["steps"] / r["total_s"]
        print(f"{name} n={d2.n} {mode:7s} steps={r['steps']} damped={r['damped']} total={r['total_s']*1e3:.1f} ms "
              f"elastic={r['elastic_s']*1e3:.1f} damping={r['damping_s']*1e3:.1f} -> {ps/1e9:.3f} G PS/s "
              f"(init {t_init:.1f} s)", flush=True)
