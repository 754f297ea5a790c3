"""Host<->device field transfer rates through the library (set_field / get_field: the pinned-ring
pipeline of csrc/cuda/hostio.cu for pageable numpy arrays), cfg2- and cfg4-sized fields."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2103_08932_b200 import dev  # noqa: E402
from paper_2103_08932_b200 import scenarios as S  # noqa: E402

for name, side in (("cfg2", 64), ("cfg2x8", 128)):
    cfg = S.cfg2(side)
    d = dev.DeviceSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"])
    n = d.n
    for field, comps in (("v", 3), ("F", 9), ("m", 1)):
        a = np.random.rand(n, comps) if comps > 1 else np.random.rand(n)
        if comps == 9:
            a = a.reshape(n, 3, 3)
        d.set(field, a)
        reps = 20
        t0 = time.perf_counter()
        for _ in range(reps):
            d.set(field, a)
        up = (time.perf_counter() - t0) / reps
        out = np.empty_like(a)
        d.get(field, out=out)
        t0 = time.perf_counter()
        for _ in range(reps):
            d.get(field, out=out)
        down = (time.perf_counter() - t0) / reps
        assert np.array_equal(out, a)
        print(f"{name} n={n} {field}: {a.nbytes/1e6:.1f} MB up {up*1e3:.3f} ms ({a.nbytes/up/1e9:.1f} GB/s) "
              f"down {down*1e3:.3f} ms ({a.nbytes/down/1e9:.1f} GB/s)", flush=True)
    del d
