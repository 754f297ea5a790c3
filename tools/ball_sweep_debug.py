"""FAST vs ORDERED vs oracle: one particle-split sweep on the falling-ball disk (2D, no clamps)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2103_08932_b200 import dev  # noqa: E402

c = O.case_setup("falling_ball")
r0 = c["r0"]
n = len(r0)
rng = np.random.RandomState(5)
for label, cons in (("no clamps", np.zeros(n, np.uint8)), ("one clamp", (np.arange(n) == 0).astype(np.uint8))):
    for vlabel, v in (("uniform v", np.tile([0.0, -0.0037], (n, 1))), ("random v", rng.normal(size=(n, 2)))):
        v = v.copy()
        v[cons == 1] = 0
        o = O.OracleSystem(r0, c["V0"], c["rho0"], c["h"], constrained=cons)
        o.set("v", v)
        o.damping_sweep("particle_split", 27950.0, 3.8e-4)
        vo = o.get("v")
        for mode in ("ordered", "fast"):
            for tiling in ("staged", "streamed"):
                d = dev.DeviceSystem(r0, c["V0"], c["rho0"], c["h"], constrained=cons)
                d.set_reduction(mode)
                d.set_sweep_tiling(tiling)
                d.set("v", v)
                d.damping_sweep("particle_split", 27950.0, 3.8e-4)
                vd = d.get("v")
                err = np.abs(vd - vo).max() / max(np.abs(vo).max(), 1e-300)
                print(f"{label:9s} {vlabel:9s} {mode:7s} {tiling:8s} max rel err {err:.3e}  spread {np.ptp(vd[:, 1]):.3e}",
                      flush=True)
