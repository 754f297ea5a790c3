#!/bin/bash
# DRAM bytes of the first 40 sweep launches on cfg4 (warm L2 between kernels), phase-by-phase vs
# blocked 12,3, bulk-store vs plain-store write-back (variant wbplain).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
o=gpurun_out/blkncu2; mkdir -p $o
for lib in default wbplain; do
  if [ $lib = default ]; then unset TLSPH_CUDA_LIB; else export TLSPH_CUDA_LIB=$PWD/paper_2103_08932_b200/lib/libtlsph_cuda_$lib.so; fi
  for b in 0 12,3; do
    TLSPH_SWEEP_BLOCK=$b timeout 300 ncu --cache-control none --clock-control none -k regex:k_sweep_fast -c 40 \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
      python tools/cfg_steps.py cfg4 --steps 0 --sweeps 1 > $o/${lib}_${b}.csv 2> $o/${lib}_${b}.err
  done
done
