#!/bin/bash
# A/B: evict-first streaming loads of slot data (default build) vs plain loads (variant nohint),
# cfg4 elastic step + sweeps, with and without the temporally blocked sweep schedule.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
o=gpurun_out/abhint; mkdir -p $o
for lib in default nohint; do
  if [ $lib = default ]; then unset TLSPH_CUDA_LIB; else export TLSPH_CUDA_LIB=$PWD/paper_2103_08932_b200/lib/libtlsph_cuda_$lib.so; fi
  echo "== $lib" >> $o/ab.log
  TLSPH_SWEEP_BLOCK=0 timeout 200 python tools/cfg_steps.py cfg4 --steps 10 --sweeps 3 >> $o/ab.log 2>&1
  for b in 0 24,6 12,3; do
    echo "-- block $b" >> $o/ab.log
    TLSPH_SWEEP_BLOCK=$b timeout 200 python tools/sweep_sizes.py cfg4 cfg5_weak --sweeps 5 >> $o/ab.log 2>&1
  done
done
