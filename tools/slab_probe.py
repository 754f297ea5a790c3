"""Linked slab sweeps on one GPU (tlsph_dev_sweep_linked): a body split into N x-slabs, each slab on
its own stream, the per-phase barrier as stream event dependencies; device time per sweep against
the undivided body. On one GPU the slabs share the SMs, so this measures the protocol's overhead,
not scaling.

  python tools/slab_probe.py [side] [sweeps] [worlds, e.g. 2,4]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2103_08932_b200 import dev, slabs  # noqa: E402
from paper_2103_08932_b200 import scenarios as S  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 64
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = S.cfg2(side)
r0, v0, h = cfg["r0"], cfg["v0"], cfg["h"]
eta, dt = cfg["eta"], cfg["fixed_dt"]
whole = dev.DeviceSystem(r0, cfg["V0"], cfg["rho0"], h)
whole.set("v", v0)
whole.damping_sweep("particle_split", eta, dt, count=2)
t1 = whole.damping_sweep("particle_split", eta, dt, count=sweeps) / sweeps
print(f"undivided {len(r0)} particles: {t1 * 1e3:.3f} ms per sweep", flush=True)
del whole  # large bodies: one copy of the state on the device at a time
for world in [int(w) for w in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["2", "3", "4"])]:
    grid, parts = slabs.decompose(r0, h, world)
    systems = [slabs.make_device_slab(grid, s, r0, cfg["V0"], cfg["rho0"], h) for s in parts]
    for s, d in zip(parts, systems):
        d.set("v", v0[s.ids])
    slabs.link_peers(systems)
    slabs.sweep_linked(systems, "particle_split", eta, dt, 2)
    t = slabs.sweep_linked(systems, "particle_split", eta, dt, sweeps) / sweeps
    print(f"{world} linked slabs on one GPU: {t * 1e3:.3f} ms per sweep ({t / t1:.2f}x undivided)", flush=True)
    del systems, d  # release the slabs before the next decomposition
