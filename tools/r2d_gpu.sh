#!/bin/bash
# Round-2d record pass (one GPU): GPU tests, the bench line, its ncu launch list, ncu --set full of
# the slot-order passes B and C (32-byte record gathers) on cfg4, the headline workload.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
o=gpurun_out/r2d; mkdir -p $o
timeout 2400 python -m pytest tests -m gpu -x -q > $o/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $o/pytest.log
python bench.py > $o/bench.json 2> $o/bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $o/launches.csv \
   python bench.py --steps 2 --warmup 1 --no-cpu --no-legs --no-e2e > $o/launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_momentum_ordered|k_deformation_rate_ordered|k_pack_v4" -s 3 -c 3 -o $o/cfg4_tl \
   python tools/cfg_steps.py cfg4 --steps 2 --sweeps 0 > $o/cfg4_tl_ncu.log 2>&1
ls -la $o
