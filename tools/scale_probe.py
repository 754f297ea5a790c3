"""Large-body probe: build cfg4 (jittered 7.8M) / cfg5-weak (15.6M) on one GPU, time init, one sweep
and a few loop steps (FAST)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08932_b200 import scenarios as S  # noqa: E402

which = sys.argv[1:] or ["cfg4", "cfg5_weak"]
for name in which:
    t0 = time.perf_counter()
    cfg = getattr(S, name)()
    t1 = time.perf_counter()
    d = S.build_device(cfg, prepare=True)
    d.set_reduction("fast")
    t2 = time.perf_counter()
    slots = d.slot_count
    el = d.damping_sweep("particle_split", cfg["eta"] / cfg["alpha"], 1e-6)
    r = d.run(S.material(), eta=cfg["eta"], alpha=cfg["alpha"], steps=20, seed=cfg["seed"])
    print(f"{name}: n={d.n} slots={slots} host gen {t1 - t0:.1f} s, device init {t2 - t1:.1f} s; "
          f"sweep {el * 1e3:.2f} ms = {2 * slots / el / 1e9:.1f} G DPU/s; 20 steps {r['total_s'] * 1e3:.1f} ms "
          f"(elastic {r['elastic_s'] * 1e3:.1f}, damping {r['damping_s'] * 1e3:.1f}, damped {r['damped']}) "
          f"-> {d.n * r['steps'] / r['total_s'] / 1e9:.3f} G PS/s", flush=True)
    del d
