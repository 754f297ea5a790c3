#!/bin/bash
# Round-2 record: full GPU suite, the default bench line, the headline's ncu launch list.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
o=gpurun_out/r2b; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > $o/gputest.log 2>&1; echo rc=$? >> $o/gputest.log
timeout 900 python bench.py > $o/bench.json 2> $o/bench.err; echo rc=$? >> $o/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $o/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-legs --no-e2e > $o/ncu_bench.log 2>&1
