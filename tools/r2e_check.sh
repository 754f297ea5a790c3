#!/bin/bash
# Round-2e: sweep times of the default build and the whole GPU suite.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/r2e
LIBS="${LIBS:-main}" bash tools/ab_sweep_libs.sh > gpurun_out/r2e/sweeps_main.log 2>&1; grep -v "^$" gpurun_out/r2e/sweeps_main.log | tail -24
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2e/pytest.log 2>&1; tail -3 gpurun_out/r2e/pytest.log
