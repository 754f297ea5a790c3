#!/bin/bash
# Round-2e: dense rows of the streamed FAST chain -- same-box A/B (TLSPH_SWEEP_DENSE=0 vs the size rule)
# and the sweep / loop / slab parity tests with dense rows forced on every body.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/r2e
for rep in 1 2; do for dm in 0 auto; do
  echo "== TLSPH_SWEEP_DENSE=$dm"
  if [ $dm = auto ]; then unset TLSPH_SWEEP_DENSE; else export TLSPH_SWEEP_DENSE=$dm; fi
  python tools/sweep_sizes.py cfg3 cfg4 cfg5_weak --sweeps 10
done; done > gpurun_out/r2e/ab_dense.log 2>&1
unset TLSPH_SWEEP_DENSE
grep -E "==|sweep" gpurun_out/r2e/ab_dense.log
TLSPH_SWEEP_DENSE=1 timeout 1500 python -m pytest tests -m gpu -x -q -k "sweep or uniform or cfg2 or loop or slab or cfg4 or cfg5" > gpurun_out/r2e/pytest_dense.log 2>&1; tail -3 gpurun_out/r2e/pytest_dense.log
