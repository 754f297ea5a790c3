"""bench.py's arms on CPU: the reference arm builds cfg4 from the oracle's own lattice and
RandomSource (no product library on its path) and must feed the oracle exactly the inputs the
GPU arm's scenario builder produces; both arms emit the same `config` dict."""
import numpy as np

import bench
from paper_2103_08932_b200 import scenarios as S


def test_reference_arm_inputs_equal_scenario_inputs():
    ref = bench.reference_cfg4_inputs()
    ours = S.cfg4()
    for k in ("r0", "v0", "constrained", "body"):
        assert np.array_equal(ref[k], ours[k]), k
    for k in ("V0", "rho0", "h", "eta", "alpha", "seed"):
        assert ref[k] == ours[k], k


def test_both_arms_share_the_config_dict():
    a = bench.cfg4_config(7_812_500, 560_132_444, 20, 5)
    b = bench.cfg4_config(7_812_500, 560_132_444, 20, 5)
    assert a == b and a["particles"] == 7_812_500 and "window" in a


def test_algorithmic_byte_model():
    # cfg3 elastic step 4.20 GB; cfg2 sweep 514.7 MB
    assert abs(bench.step_bytes(640_000, 48_611_784) / 1e9 - 4.198) < 0.01
    assert abs(bench.sweep_bytes(20_026_056, 262_144) / 1e6 - 514.7) < 0.5
