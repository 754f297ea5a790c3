"""Cell-tiled FAST pass B (TLSPH_TL_TILED=4|8) against the oracle: a jittered 3D block (n >= 65,536,
so the untiled FAST path runs the slot-order kernels) and a 2D plate, 8 loop steps each; prints the
relative L2 of v, r, F against the oracle and the elastic step time. Run once per setting:
  TLSPH_TL_TILED=4 python tools/tiled_check.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2103_08932_b200 import dev  # noqa: E402
from paper_2103_08932_b200 import scenarios as S  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def case(r0, dp, cons, steps=8):
    dim = r0.shape[1]
    h = 1.3 * dp
    n = len(r0)
    v = 0.02 * (dev.random_uniforms(7, n * dim).reshape(n, dim) - 0.5)
    v[cons == 1] = 0.0
    g = np.zeros((n, dim))
    g[:, 1] = -9.81
    mat = S.material()
    d = dev.DeviceSystem(r0, dp ** dim, S.RHO0, h, constrained=cons)
    d.set_reduction("fast")
    d.set("v", v)
    d.set("body", g)
    d.prepare(mat)
    r = d.run(mat, eta=S.eta_for(h), alpha=0.3, steps=steps, seed=1)
    o = O.OracleSystem(r0, dp ** dim, S.RHO0, h, constrained=cons)
    o.set_material(S.E_MOD, S.NU, S.RHO0)
    o.set("v", v)
    o.set("body", g)
    o.prepare(threads=O.openmp_threads())
    ro = o.run(eta=S.eta_for(h), alpha=0.3, seed=1, steps=steps, threads=O.openmp_threads())
    print(f"n={n} dim={dim} tiled={os.environ.get('TLSPH_TL_TILED', '0')}: steps {r['steps']} damped {r['damped']}/"
          f"{ro['damped']} rel v {rel(d.get('v'), o.get('v')):.2e} r {rel(d.get('r'), o.get('r')):.2e} "
          f"F {rel(d.get('F'), o.get('F')):.2e} elastic {r['elastic_s'] / r['steps'] * 1e3:.3f} ms/step", flush=True)


dp = 0.01
r0, _ = S.box_lattice([0, 0, 0], [0.5, 0.5, 0.3], dp)
u = dev.random_uniforms(3, r0.size).reshape(r0.shape)
r0 = np.ascontiguousarray(r0 + (2 * u - 1) * 0.4 * dp)
case(r0, dp, (r0[:, 0] < 3 * dp).astype(np.uint8))
r2, _ = S.box_lattice([0, 0], [0.6, 0.1], 0.0025)
case(r2, 0.0025, (r2[:, 0] < 4 * 0.0025).astype(np.uint8))
