"""cfg2 pairwise-split sweeps (ORDERED = FAST, bit-exact), for timing and an ncu capture of one phase."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08932_b200 import scenarios as S  # noqa: E402

sweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = S.cfg2()
d = S.build_device(cfg, prepare=False)
eta_t = cfg["eta"] / cfg["alpha"]
d.damping_sweep("pairwise_split", eta_t, cfg["fixed_dt"])
el = d.damping_sweep("pairwise_split", eta_t, cfg["fixed_dt"], count=sweeps) / sweeps
print(f"pairwise cfg2: {el * 1e3:.3f} ms/sweep, {2 * d.slot_count / el / 1e9:.2f} G DPU/s", flush=True)
