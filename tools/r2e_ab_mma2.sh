#!/bin/bash
# Round-2e A/B: warp sum of the FAST chain by two MMAs and no shuffle (-DTLSPH_SWEEP_MMA_SUM=2).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/r2e
LIBS="main mma2" bash tools/ab_sweep_libs.sh > gpurun_out/r2e/ab_mma2.log 2>&1; grep -v "^$" gpurun_out/r2e/ab_mma2.log | tail -40
TLSPH_CUDA_LIB=$PWD/paper_2103_08932_b200/lib/libtlsph_cuda_mma2.so timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sweep or uniform or cfg2 or loop" > gpurun_out/r2e/pytest_mma2.log 2>&1; tail -3 gpurun_out/r2e/pytest_mma2.log
