#!/bin/bash
# DRAM bytes per launch of the temporally blocked vs phase-by-phase sweep (warm L2 between
# kernels: --cache-control none), cfg4 and cfg5-weak, one sweep each.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
o=gpurun_out/blkncu; mkdir -p $o
for cfg in cfg4 cfg5_weak; do
for b in 0 24,6 12,3; do
  TLSPH_SWEEP_BLOCK=$b timeout 900 ncu --cache-control none --clock-control none -k regex:k_sweep_fast -c 120 \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --csv \
    python tools/cfg_steps.py $cfg --steps 0 --sweeps 1 > $o/${cfg}_${b}.csv 2> $o/${cfg}_${b}.err
done
done
