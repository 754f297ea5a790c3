"""tlsph_sim_run end to end against the oracle's run of the same built-in case.

The C ABI call (libtlsph.so.1: tlsph_sim_create with config overrides, tlsph_sim_run) writes
probe.csv and report.json (runner.cpp:393-413, 422-488); the oracle builds the same case
(oracle.case_setup, cases.cpp:160-231), initialises it as runner.cpp:299-313 does and runs the loop
of :341-391 with the probe series of :328,378-395. Linear Kirchhoff (falling_ball, with its
contact plane) in ORDERED mode is bit-exact arithmetic, so its probe.csv must be byte-identical
(the reference pins byte-identical probe files, tests/test_runner.cpp:176-200); neo-Hookean
cases (ORDERED: log() within an ulp; FAST: lane-parallel sums) agree within 1e-10.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2103_08932_b200", "lib", "libtlsph.so.1")


def sim_run(overrides):
    L = C.CDLL(LIB)
    L.tlsph_sim_create.argtypes = [C.c_char_p, C.POINTER(C.c_char_p), C.c_size_t, C.POINTER(C.c_void_p)]
    L.tlsph_sim_run.argtypes = [C.c_void_p]
    L.tlsph_sim_destroy.argtypes = [C.c_void_p]
    L.tlsph_sim_step_count.argtypes = [C.c_void_p]
    L.tlsph_sim_step_count.restype = C.c_uint64
    L.tlsph_sim_damped_step_count.argtypes = [C.c_void_p]
    L.tlsph_sim_damped_step_count.restype = C.c_uint64
    L.tlsph_last_error.restype = C.c_char_p
    arr = (C.c_char_p * len(overrides))(*[o.encode() for o in overrides])
    sim = C.c_void_p()
    st = L.tlsph_sim_create(None, arr, len(overrides), C.byref(sim))
    assert st == 0, L.tlsph_last_error().decode()
    try:
        st = L.tlsph_sim_run(sim)
        assert st == 0, L.tlsph_last_error().decode()
        return int(L.tlsph_sim_step_count(sim)), int(L.tlsph_sim_damped_step_count(sim))
    finally:
        L.tlsph_sim_destroy(sim)


def read_probe(path):
    with open(path, "rb") as fh:
        raw = fh.read().decode()
    rows = [list(map(float, line.split(","))) for line in raw.strip().split("\n")[1:]]
    return raw, np.array(rows)


CASES = [
    ("falling_ball", 0, 0.2, "ordered", "bytes"),  # free fall (the floor is reached at t ~ 0.226 s)
    ("falling_ball", 0, 0.2, "fast", 1e-10),
    ("bending_cantilever", 0, 0.03, "ordered", 1e-10),
    ("bending_cantilever", 0, 0.03, "fast", 1e-10),
    ("twisting_cantilever", 6, 0.03, "ordered", 1e-10),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,res,end,mode,bar", CASES, ids=lambda x: str(x))
def test_sim_run_probe_series_matches_oracle(tmp_path, name, res, end, mode, bar):
    out = str(tmp_path / "out")
    ov = [f"case={name}", f"end_time={end}", f"output.dir={out}", "output.snapshots=none", f"gpu.reduction={mode}",
          "output.interval=0.005"]
    if res:
        ov.append(f"resolution={res}")
    steps, damped = sim_run(ov)
    raw, got = read_probe(os.path.join(out, "probe.csv"))
    want, r, _ = O.run_case(name, res, end_time=end, interval=0.005)
    assert steps == r["steps"] and damped == r["damped"], (steps, damped, r["steps"], r["damped"])
    assert got.shape == want.shape, (got.shape, want.shape)
    assert damped > 0 and len(want) >= 5
    if bar == "bytes":
        assert raw == O.probe_csv(want, want.shape[1] - 1), "probe.csv differs from the oracle's bytes"
    else:
        assert np.allclose(got[:, 0], want[:, 0], rtol=1e-12, atol=0.0)
        scale = np.abs(want[:, 1:]).max()
        err = np.abs(got[:, 1:] - want[:, 1:]).max() / scale
        assert err <= bar, f"probe displacement differs by {err:.3e} of its scale"
    rep = json.load(open(os.path.join(out, "report.json")))
    assert rep["steps"] == r["steps"] and rep["damped_steps"] == r["damped"]
    assert np.allclose(rep["final_probe_u"], want[-1, 1:], rtol=1e-9, atol=1e-14 * scale if bar != "bytes" else 0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["ordered", "fast"])
def test_sim_run_fails_like_the_oracle_at_floor_contact(tmp_path, mode):
    """Past t ~ 0.226 s the ball's bottom rows meet the penalty floor (stiffness K, cases.cpp:207-212)
    and an element inverts; the reference path (integrator.cpp:101-102 via update_density) throws
    InvertedElement naming the lowest such particle. tlsph_sim_run must fail the same way: status
    TLSPH_ERR_INVERTED_ELEMENT with the oracle's message."""
    with pytest.raises(O.OracleError) as oe:
        O.run_case("falling_ball", 0, end_time=0.3)
    L = C.CDLL(LIB)
    L.tlsph_sim_create.argtypes = [C.c_char_p, C.POINTER(C.c_char_p), C.c_size_t, C.POINTER(C.c_void_p)]
    L.tlsph_sim_run.argtypes = [C.c_void_p]
    L.tlsph_sim_destroy.argtypes = [C.c_void_p]
    L.tlsph_last_error.restype = C.c_char_p
    ov = ["case=falling_ball", "end_time=0.3", "output.dir=", f"gpu.reduction={mode}"]
    arr = (C.c_char_p * len(ov))(*[o.encode() for o in ov])
    sim = C.c_void_p()
    assert L.tlsph_sim_create(None, arr, len(ov), C.byref(sim)) == 0
    try:
        st = L.tlsph_sim_run(sim)
        msg = L.tlsph_last_error().decode()
    finally:
        L.tlsph_sim_destroy(sim)
    assert st == 4, (st, msg)  # TLSPH_ERR_INVERTED_ELEMENT
    assert msg == oe.value.message, (msg, oe.value.message)


def test_oracle_cases_follow_the_reference_geometry():
    """cases.cpp:160-231 restated: particle counts (18 x 6 x 6 cantilever rows as in
    tests/test_runner.cpp:172), clamp layers, probe targets, free fall of the ball before contact."""
    c = O.case_setup("bending_cantilever")
    assert len(c["r0"]) == 18 * 6 * 6
    assert int(c["constrained"].sum()) == 3 * 6 * 6
    dp = 0.016 / 6
    assert np.allclose(np.abs(c["r0"][c["probe"]]), [0.04 - 0.5 * dp, 0.5 * dp, 0.5 * dp], rtol=1e-12)
    b = O.case_setup("falling_ball")
    assert b["contact"] is not None and b["contact"][2] == O.material(5e5, 0.45, 1000.0, "linear_kirchhoff")["K"]
    assert np.allclose(b["r0"][b["probe"]], [0.0, 0.75])
    p, r, _ = O.run_case("falling_ball", end_time=0.05, interval=0.01)
    # no contact before the bottom reaches the floor: u_y = -g t^2 / 2 to rounding
    assert np.allclose(p[:, 2], -0.5 * 9.8 * p[:, 0] ** 2, rtol=1e-9, atol=1e-15)
