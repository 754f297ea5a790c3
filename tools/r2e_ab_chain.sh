#!/bin/bash
# Round-2e A/B of chain variants: LIBS / CFGS as tools/ab_sweep_libs.sh; then the sweep parity tests on each variant.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/r2e
bash tools/ab_sweep_libs.sh > gpurun_out/r2e/ab_chain.log 2>&1; grep -v "^$" gpurun_out/r2e/ab_chain.log | tail -60
for L in $TESTLIBS; do
  TLSPH_CUDA_LIB=$PWD/paper_2103_08932_b200/lib/libtlsph_cuda_$L.so timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sweep or uniform or cfg2 or loop" > gpurun_out/r2e/pytest_$L.log 2>&1; echo $L; tail -2 gpurun_out/r2e/pytest_$L.log
done
