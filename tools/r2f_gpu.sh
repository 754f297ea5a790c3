#!/bin/bash
# Round-2f (final) record pass on one GPU: smoke, the GPU suite, the bench line and its ncu launch list.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
o=gpurun_out/r2f; mkdir -p $o
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $o/smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q > $o/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $o/pytest.log
python bench.py > $o/bench.json 2> $o/bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $o/launches.csv \
   python bench.py --steps 2 --warmup 1 --no-cpu --no-legs --no-e2e > $o/launch_run.log 2>&1
ls -la $o
