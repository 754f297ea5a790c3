"""Falling-ball FAST vs ORDERED divergence probe: the oracle's case on the device loop, no contact
(t < 0.2 s), max |F - I| and max velocity spread after K steps in each mode."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2103_08932_b200 import dev  # noqa: E402

c = O.case_setup("falling_ball")
sp = c["spec"]

for mode in ("ordered", "fast"):
    for contact in (False,):
        for steps in (1, 2, 5, 20, 100, 400):
            d = dev.DeviceSystem(c["r0"], c["V0"], c["rho0"], c["h"], constrained=c["constrained"])
            d.set_reduction(mode)
            d.set("body", c["body"])
            m = dev.Material.from_young_poisson(sp["E"], sp["nu"], sp["rho0"], sp["model"])
            d.prepare(m)
            try:
                r = d.run(m, eta=c["eta"], alpha=c["alpha"], steps=steps, seed=0)
                F = d.get("F")
                v = d.get("v")
                eye = np.eye(2)
                print(mode, steps, "damped", r["damped"], "max|F-I|", np.abs(F - eye).max(), "v spread",
                      np.ptp(v[:, 1]), "t", r["t"], flush=True)
            except Exception as ex:
                print(mode, steps, "ERR", ex, flush=True)
