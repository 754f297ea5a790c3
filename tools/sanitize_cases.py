"""Small bodies through every device path, for compute-sanitizer (memcheck / racecheck / synccheck):

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py [small|large]

small: 3D lattice (~5k particles) and a 2D plate -- staged sweeps (FAST + ORDERED, particle and
pairwise split), the streamed sweep (TLSPH_SWEEP_STREAM=1 in the environment), explicit damping,
the TL-SPH operators and a 6-step device loop with graphs and the per-step cell rebuild.
large: a 70k-particle jittered block (the one-thread slot-order TL-SPH passes, n >= 65,536) for a
few loop steps. Every case's result is checked finite; sanitizer findings are in its own report.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08932_b200 import dev  # noqa: E402
from paper_2103_08932_b200 import scenarios as S  # noqa: E402


def body(lo, hi, dp, jitter=0.0, seed=3):
    r0, _ = S.box_lattice(lo, hi, dp)
    n, dim = r0.shape
    if jitter:
        u = dev.random_uniforms(seed, n * dim).reshape(n, dim)
        r0 = np.ascontiguousarray(r0 + (2.0 * u - 1.0) * jitter * dp)
    v = -0.01 + 0.02 * dev.random_uniforms(seed + 1, n * dim).reshape(n, dim)
    cons = (r0[:, 0] < 3 * dp).astype(np.uint8)
    v[cons == 1] = 0.0
    g = np.zeros((n, dim))
    g[:, 1] = -S.GRAVITY
    return r0, v, cons, g


def run_case(r0, v, cons, g, dp, modes=("fast", "ordered"), steps=6):
    dim = r0.shape[1]
    h = 1.3 * dp
    mat = S.material()
    for mode in modes:
        d = dev.DeviceSystem(r0, dp ** dim, S.RHO0, h, constrained=cons)
        d.set("v", v)
        d.set("body", g)
        d.set_reduction(mode)
        d.prepare(mat)
        eta = S.eta_for(h)
        dt = d.stable_dt(mat)
        for scheme in ("particle_split", "pairwise_split"):
            d.damping_sweep(scheme, eta / 0.2, dt, count=2)
        d.explicit_damping_accel(eta)
        d.verlet_step(mat, dt)
        d.set_resort(True)
        r = d.run(mat, eta=eta, alpha=0.5, steps=steps, seed=0)
        vv = d.get("v")
        assert np.isfinite(vv).all(), "non-finite velocities"
        print(f"  n={d.n} dim={dim} mode={mode} steps={r['steps']} damped={r['damped']} ok", flush=True)
        d.close()


which = sys.argv[1] if len(sys.argv) > 1 else "small"
print(f"sanitize_cases {which} TLSPH_SWEEP_STREAM={os.environ.get('TLSPH_SWEEP_STREAM', 'auto')}", flush=True)
if which == "small":
    dp = 0.01
    run_case(*body([0, 0, 0], [0.2, 0.16, 0.12], dp, jitter=0.3), dp)
    dp2 = 0.0025
    run_case(*body([0, 0], [0.2, 0.05], dp2), dp2)
else:
    dp = 0.01
    run_case(*body([0, 0, 0], [0.48, 0.4, 0.4], dp, jitter=0.4), dp, modes=("fast",), steps=3)
print("sanitize_cases done", flush=True)
