"""bench.py's arms on CPU: the reference arm builds cfg4 from the oracle's own lattice and
RandomSource (no product library on its path) and must feed the oracle exactly the inputs the
GPU arm's scenario builder produces; both arms emit the same `config` dict."""
import os

import numpy as np
import pytest

import bench
from paper_2103_08932_b200 import scenarios as S


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


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


@pytest.mark.gpu
def test_bench_n2_protocol_through_the_c_group(tmp_path):
    """bench.py --gpus 2 under torchrun (both ranks on one device: TLSPH_BENCH_ONE_DEVICE=1, the
    protocol only, not a timing): one JSON line from rank 0 with the sharded cfg5 value driven by
    the C entry point (tlsph_dev_group_run)."""
    import json
    import socket
    import subprocess
    import sys

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, TLSPH_BENCH_ONE_DEVICE="1")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--steps", "2", "--warmup", "1", "--scale-layers", "12", "--scale-sweeps", "3"],
                         capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 2
    assert "tlsph_dev_group_run" in d["config"]["driver"]
    assert d["sweep"]["value"] > 0
