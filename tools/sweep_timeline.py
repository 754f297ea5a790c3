"""Per-cell stage timeline of one colour phase of the cfg2 sweep (debug build with %globaltimer stamps).

    make -C paper_2103_08932_b200/csrc timing
    TLSPH_CUDA_LIB=paper_2103_08932_b200/lib/libtlsph_cuda_timing.so python tools/sweep_timeline.py
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08932_b200 import dev  # noqa: E402
from paper_2103_08932_b200 import scenarios as S  # noqa: E402

cfg = S.cfg2()
d = S.build_device(cfg, prepare=False)
eta_t = cfg["eta"] / cfg["alpha"]
for _ in range(3):
    d.damping_sweep("particle_split", eta_t, cfg["fixed_dt"])
L = dev.lib()
L.tlsph_debug_sweep_stamps.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
ncell = 579
buf = (C.c_ulonglong * (8 * ncell))()
n = L.tlsph_debug_sweep_stamps(buf, ncell)
st = np.array(buf[: 8 * n], dtype=np.float64).reshape(n, 8)
order = [0, 6, 1, 2, 3, 4, 5]
names = ["start", "indices-loaded", "tma-issued", "tma-landed", "staged", "chain-done", "written"]
st = st[:, order]
t0 = st[:, 0].min()
rel = (st - t0) / 1e3  # microseconds
print(f"cells {n}; phase span {rel[:, -1].max():.2f} us")
for k, name in enumerate(names):
    print(f"{name:15s} min {rel[:, k].min():7.2f}  median {np.median(rel[:, k]):7.2f}  max {rel[:, k].max():7.2f} us")
dur = np.diff(rel, axis=1)
for k in range(len(names) - 1):
    print(f"{names[k]:>15s} -> {names[k + 1]:15s} median {np.median(dur[:, k]):6.2f} us  max {dur[:, k].max():6.2f}")

