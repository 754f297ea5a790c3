"""The paper's Table 1 workload: damping time of the bending cantilever at
h/dp = 12 to t = 2 s with the particle-split scheme, alpha = 1.0 and 0.2, through tlsph_sim_run
(the reference's built-in case; note its geometry is 0.04 x 0.016 m, cases.cpp:81-82, not the
paper's 0.1 x 0.04) -- and the oracle (the reference path on the host cores) on the same case.
Prints one JSON line per run with the phase seconds (runner.cpp's neighbor / elastic / damping).

  python tools/paper_table1.py [--oracle]
"""
import ctypes as C
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2103_08932_b200", "lib",
                   "libtlsph.so.1")


def sim(overrides):
    L = C.CDLL(LIB)
    L.tlsph_sim_create.argtypes = [C.c_char_p, C.POINTER(C.c_char_p), C.c_size_t, C.POINTER(C.c_void_p)]
    L.tlsph_sim_run.argtypes = [C.c_void_p]
    L.tlsph_sim_destroy.argtypes = [C.c_void_p]
    L.tlsph_sim_phase_seconds.argtypes = [C.c_void_p, C.c_char_p]
    L.tlsph_sim_phase_seconds.restype = C.c_double
    L.tlsph_sim_step_count.argtypes = [C.c_void_p]
    L.tlsph_sim_step_count.restype = C.c_uint64
    L.tlsph_sim_damped_step_count.argtypes = [C.c_void_p]
    L.tlsph_sim_damped_step_count.restype = C.c_uint64
    L.tlsph_last_error.restype = C.c_char_p
    arr = (C.c_char_p * len(overrides))(*[o.encode() for o in overrides])
    h = C.c_void_p()
    assert L.tlsph_sim_create(None, arr, len(overrides), C.byref(h)) == 0, L.tlsph_last_error()
    try:
        assert L.tlsph_sim_run(h) == 0, L.tlsph_last_error()
        return {k: L.tlsph_sim_phase_seconds(h, k.encode()) for k in ("neighbor", "elastic", "damping", "total")} | {
            "steps": int(L.tlsph_sim_step_count(h)), "damped": int(L.tlsph_sim_damped_step_count(h))}
    finally:
        L.tlsph_sim_destroy(h)


paper = {1.0: {"serial_s": 32.82, "parallel_6core_s": 11.61}, 0.2: {"serial_s": 6.66, "parallel_6core_s": 2.38}}
for alpha in (1.0, 0.2):
    for mode in ("fast", "ordered"):
        r = sim(["case=bending_cantilever", "resolution=12", "end_time=2.0", f"damping.alpha={alpha}", "output.dir=",
                 f"gpu.reduction={mode}"])
        print(json.dumps({"run": f"gpu-{mode}", "alpha": alpha, **r, "paper_damping_s": paper[alpha]}), flush=True)
if "--oracle" in sys.argv:
    import time

    from oracle import oracle as O

    for alpha in (1.0, 0.2):
        c = O.case_setup("bending_cantilever", 12)
        sp = c["spec"]
        threads = O.openmp_threads()
        o = O.OracleSystem(c["r0"], c["V0"], c["rho0"], c["h"], constrained=c["constrained"])
        o.set_material(sp["E"], sp["nu"], sp["rho0"], sp["model"])
        o.set("body", c["body"])
        o.prepare(threads=threads)
        t0 = time.perf_counter()
        r = o.run(eta=c["eta"], alpha=alpha, seed=0, steps=1 << 62, end_time=2.0, threads=threads)
        print(json.dumps({"run": "oracle", "alpha": alpha, "threads": threads, "steps": r["steps"],
                          "damped": r["damped"], "elastic": r["elastic_s"], "damping": r["damping_s"],
                          "total": time.perf_counter() - t0, "paper_damping_s": paper[alpha]}), flush=True)
