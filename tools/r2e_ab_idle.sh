cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/r2e
LIBS="noidle main" bash tools/ab_sweep_libs.sh > gpurun_out/r2e/ab_idle.log 2>&1; cat gpurun_out/r2e/ab_idle.log | grep -v "^$" | tail -40
timeout 1200 python -m pytest tests -m gpu -x -q -k "sweep or slab or uniform or cfg2 or loop" > gpurun_out/r2e/pytest_sweep.log 2>&1; tail -3 gpurun_out/r2e/pytest_sweep.log
