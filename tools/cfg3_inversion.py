"""BASELINE cfg3 at full resolution (640,000 particles) to its end: the device loop (ORDERED and FAST)
and the oracle (the reference path, OpenMP on every host core) run the KE-stop loop of
runner.cpp:341-391 until it stops -- on the KE criterion or, as the soft beam does, on the
reference's InvertedElement error (integrator.cpp:101-102). Prints one JSON line per run: steps,
t, stop reason. Long: the oracle needs ~1 h of 16 cores.

  python tools/cfg3_inversion.py [--skip-oracle]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_08932_b200 import scenarios as S  # noqa: E402

cfg = S.cfg3()
out = {}
for mode in ("ordered", "fast"):
    d = S.build_device(cfg, prepare=True)
    d.set_reduction(mode)
    t0 = time.perf_counter()
    try:
        r = d.run(S.material(), eta=cfg["eta"], alpha=cfg["alpha"], steps=200000, seed=cfg["seed"], ke_stop=True,
                  ke_ratio=1e-8)
        rec = {"run": f"gpu-{mode}", "steps": r["steps"], "t": r["t"], "stop": "ke" if r["stopped_on_ke"] else "cap"}
    except Exception as e:
        steps, t = d.last_run()
        rec = {"run": f"gpu-{mode}", "steps": steps, "t": t, "stop": str(e)}
    rec["wall_s"] = time.perf_counter() - t0
    print(json.dumps(rec), flush=True)
    del d
if "--skip-oracle" not in sys.argv:
    from oracle import oracle as O  # the reference path (checker)

    threads = O.openmp_threads()
    o = O.OracleSystem(cfg["r0"], cfg["V0"], cfg["rho0"], cfg["h"], constrained=cfg["constrained"])
    o.set_material(S.E_MOD, S.NU, S.RHO0)
    o.set("v", cfg["v0"])
    o.set("body", cfg["body"])
    o.prepare(threads=threads)
    t0 = time.perf_counter()
    done = 0
    rec = None
    # chunks of 2000 steps (resume keeps the damping stream, t and the step count)
    while done < 200000:
        try:
            r = o.run(eta=cfg["eta"], alpha=cfg["alpha"], seed=cfg["seed"], steps=done + 2000, threads=threads,
                      resume=done > 0)
            done = r["steps"]
            ke = o.kinetic_energy()
            print(json.dumps({"run": "oracle-progress", "steps": done, "t": r["t"], "ke": ke,
                              "wall_s": time.perf_counter() - t0}), flush=True)
        except Exception as e:
            steps, t = o.last_run()
            rec = {"run": "oracle", "steps": steps, "t": t, "stop": str(e), "threads": threads,
                   "wall_s": time.perf_counter() - t0}
            break
    print(json.dumps(rec), flush=True)
