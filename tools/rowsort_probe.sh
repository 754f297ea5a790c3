#!/bin/bash
# A/B: interleaved TL-SPH slot rows in reference order vs ascending neighbour index (TLSPH_TL_ROWSORT=1).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
o=gpurun_out/rowsort; mkdir -p $o
for rs in 0 1 0 1; do
  echo "== rowsort $rs" >> $o/ab.log
  TLSPH_TL_ROWSORT=$rs timeout 200 python tools/cfg_steps.py cfg4 --steps 12 --sweeps 0 >> $o/ab.log 2>&1
  TLSPH_TL_ROWSORT=$rs timeout 200 python tools/cfg_steps.py cfg3 --steps 50 --sweeps 0 >> $o/ab.log 2>&1
done
