"""Steps to the kinetic-energy stop (KE < ratio x peak KE, after the peak) of a cfg3-shaped beam at
reduced resolution, ORDERED and FAST on the GPU, and the oracle's final state at the ORDERED count.

  python tools/ke_stop_probe.py [scale] [ratio ...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2103_08932_b200 import scenarios as S  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 4
ratios = [float(x) for x in sys.argv[2:]] or [1e-3, 1e-6, 1e-8]
cfg = S.cfg3(scale=scale)
for ratio in ratios:
    res = {}
    for mode in ("ordered", "fast"):
        d = S.build_device(cfg, prepare=True)
        d.set_reduction(mode)
        t0 = time.perf_counter()
        try:
            r = d.run(S.material(), eta=cfg["eta"], alpha=cfg["alpha"], steps=2_000_000, seed=cfg["seed"],
                      ke_stop=True, ke_ratio=ratio)
        except Exception as e:  # the reference stops with the same error kinds
            steps, t = d.last_run()
            print(f"n={d.n} ratio={ratio:g} {mode:7s}: stopped by '{e}' after {steps} steps, t = {t:.6g} s "
                  f"({time.perf_counter() - t0:.1f} s)", flush=True)
            continue
        res[mode] = r
        print(f"n={d.n} ratio={ratio:g} {mode:7s}: steps {r['steps']} damped {r['damped']} stopped {r['stopped_on_ke']} "
              f"peak KE {r['peak_ke']:.6e} final {r['final_ke']:.6e} ({time.perf_counter() - t0:.1f} s)", flush=True)
