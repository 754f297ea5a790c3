"""Per-cell stage timeline of one colour phase of a sweep (debug build with %globaltimer stamps).

    make -C paper_2103_08932_b200/csrc timing
    TLSPH_CUDA_LIB=paper_2103_08932_b200/lib/libtlsph_cuda_timing.so python tools/sweep_timeline.py [cfg2|cfg3|cfg4|cfg5_weak]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08932_b200 import dev  # noqa: E402
from paper_2103_08932_b200 import scenarios as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = getattr(S, name)()
d = S.build_device(cfg, prepare=False)
eta_t = cfg["eta"] / cfg["alpha"]
for _ in range(3):
    d.damping_sweep("particle_split", eta_t, cfg["fixed_dt"] or 1e-5)
L = dev.lib()
L.tlsph_debug_sweep_stamps.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
SLOTS = 10
ncell = 579 if name == "cfg2" else 1 << 16
buf = (C.c_ulonglong * (SLOTS * ncell))()
n = L.tlsph_debug_sweep_stamps(buf, ncell)
st = np.array(buf[: SLOTS * n], dtype=np.float64).reshape(n, SLOTS)
ghz = float(os.environ.get("SM_GHZ", "1.965"))
start_us = (st[:, 0] - st[:, 0].min()) / 1e3
cyc = st[:, 1:8] - st[:, 1:2]  # clock64 relative to each cell's own start
nps = st[:, 8]
names = ["start", "indices", "bulk issued", "rows issued", "tma landed", "chain done", "written"]
# the stamp table is indexed by CTA and reused by every phase: keep the last phase's CTAs (CTA 0
# starts first; entries of earlier, larger phases are older)
live = (st[:, 7] > 0) & (st[:, 0] >= st[0, 0] - 5e3)
st, start_us, cyc, nps = st[live], start_us[live], cyc[live], nps[live]
n = int(live.sum())
start_us = start_us - start_us.min()
end_us = start_us + cyc[:, -1] / (ghz * 1e3)
print(f"cells {n}; CTA start spread {start_us.max():.2f} us; phase span {end_us.max():.2f} us "
      f"(median end {np.median(end_us):.2f})")
dur = np.diff(cyc, axis=1)
for k in range(len(names) - 1):
    print(f"{names[k]:>12s} -> {names[k + 1]:12s} median {np.median(dur[:, k]):7.0f} cyc "
          f"({np.median(dur[:, k]) / ghz:6.0f} ns)  max {dur[:, k].max():7.0f} cyc")
bar = st[:, 9] - st[:, 1]
print(f"  (indices -> barrier initialised: median {np.median(bar - cyc[:, 1]):.0f} cyc)")
chain = dur[:, 4]
ok = nps > 0
print(f"chain per particle: median {np.median(chain[ok] / nps[ok]):.0f} cycles (np median {np.median(nps[ok]):.0f}, "
      f"max {nps.max():.0f}); by np:")
task = cyc[:, -1]
print(f"task total: median {np.median(task):.0f} cyc ({np.median(task) / ghz / 1e3:.2f} us); sum over tasks / span = "
      f"{task.sum() / ghz / 1e3 / max(end_us.max(), 1e-9):.1f} concurrent tasks")
for v in sorted(set(nps[ok].astype(int))):
    m = nps == v
    print(f"  np {v:3d}: {m.sum():4d} cells, chain {np.median(chain[m]):7.0f} cyc, end {np.median(end_us[m]):6.2f} us")
