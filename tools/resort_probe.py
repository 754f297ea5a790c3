"""Cost of BASELINE cfg4's per-step re-sort: the jittered 7.8 M-particle block's device loop (FAST,
alpha 0.1) with and without the current-position cell rebuild every step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08932_b200 import scenarios as S  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
cfg = S.cfg4()
d = S.build_device(cfg, prepare=True)
d.set_reduction("fast")
for resort in (False, True, False, True):
    d.set_resort(resort)
    r = d.run(S.material(), eta=cfg["eta"], alpha=cfg["alpha"], steps=steps, seed=cfg["seed"])
    print(f"cfg4 n={d.n} resort={resort}: {r['total_s'] / r['steps'] * 1e3:.3f} ms per step "
          f"({d.n * r['steps'] / r['total_s'] / 1e9:.3f} G PS/s, damped {r['damped']})", flush=True)
