#!/bin/bash
# Round-2e record pass (one GPU): the bench line, its ncu launch list, ncu --set full of one
# streamed sweep phase on cfg4 and cfg5-weak and one staged phase on cfg2 (two-MMA warp sum, folded
# rate, unrolled pipeline).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
o=gpurun_out/r2e; mkdir -p $o
python bench.py > $o/bench.json 2> $o/bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $o/launches.csv \
   python bench.py --steps 2 --warmup 1 --no-cpu --no-legs --no-e2e > $o/launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_fast -s 30 -c 1 -o $o/cfg4_sweep \
   python tools/cfg_steps.py cfg4 --steps 0 --sweeps 1 > $o/cfg4_sweep_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_sweep_fast -s 30 -c 1 -o $o/cfg5w_sweep \
   python tools/cfg_steps.py cfg5_weak --steps 0 --sweeps 1 > $o/cfg5w_sweep_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_fast -s 30 -c 1 -o $o/cfg2_sweep \
   python tools/cfg_steps.py cfg2 --steps 0 --sweeps 1 > $o/cfg2_sweep_ncu.log 2>&1
ls -la $o
