#!/bin/bash
# The dataflow (temporally blocked) sweep: bitwise tests, then cfg4 / cfg5-weak sweep times over (W, k).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
o=gpurun_out/flow; mkdir -p $o
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "blocked or tiling" > $o/test.log 2>&1; echo rc=$? >> $o/test.log
grep -q "rc=0" $o/test.log || exit 0
for b in 0 auto 24,6 12,3 16,4 8,2 32,8; do
  if [ $b = auto ]; then unset TLSPH_SWEEP_BLOCK; else export TLSPH_SWEEP_BLOCK=$b; fi
  echo "== $b" >> $o/sizes.log
  timeout 240 python tools/sweep_sizes.py cfg4 cfg5_weak --sweeps 5 >> $o/sizes.log 2>&1; echo "rc=$?" >> $o/sizes.log
done
