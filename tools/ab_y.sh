#!/bin/bash
# A/B of the FAST update's Y form (TLSPH_Y_FORM variants): cfg2 / cfg4 / cfg5-weak sweep times.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
o=gpurun_out/aby; mkdir -p $o
for lib in ylate prev ylate prev; do
  if [ $lib = default ]; then unset TLSPH_CUDA_LIB; else export TLSPH_CUDA_LIB=$PWD/paper_2103_08932_b200/lib/libtlsph_cuda_$lib.so; fi
  echo "== $lib" >> $o/ab.log
  timeout 300 python tools/sweep_sizes.py cfg2 cfg4 cfg5_weak --sweeps 10 >> $o/ab.log 2>&1
done
