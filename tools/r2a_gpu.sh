#!/bin/bash
# Round-2 profiling pass (one GPU): compute-sanitizer over the small/large cases and the IPC slab
# tests, the cfg4 launch list, ncu --set full of pass B / pass C / one streamed sweep phase on cfg4.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
o=gpurun_out/r2a; mkdir -p $o
CS="compute-sanitizer --print-limit 50 --error-exitcode 9"
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool python tools/sanitize_cases.py small > $o/san_${tool}_small.log 2>&1; echo "rc=$?" >> $o/san_${tool}_small.log
  TLSPH_SWEEP_STREAM=1 timeout 900 $CS --tool $tool python tools/sanitize_cases.py small > $o/san_${tool}_small_stream.log 2>&1; echo "rc=$?" >> $o/san_${tool}_small_stream.log
done
timeout 900 $CS --tool memcheck python tools/sanitize_cases.py large > $o/san_memcheck_large.log 2>&1; echo "rc=$?" >> $o/san_memcheck_large.log
timeout 900 $CS --tool memcheck --target-processes all python -m pytest tests/test_slabs.py -q -x -m gpu -k "ipc and 2-2" > $o/san_memcheck_ipc.log 2>&1; echo "rc=$?" >> $o/san_memcheck_ipc.log
timeout 900 $CS --tool racecheck --target-processes all python -m pytest tests/test_slabs.py -q -x -m gpu -k "ipc_slabs_equal and 2-2" > $o/san_racecheck_ipc.log 2>&1; echo "rc=$?" >> $o/san_racecheck_ipc.log
timeout 600 python tools/cfg_steps.py cfg4 --steps 5 --sweeps 2 --resort > $o/cfg4_plain.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $o/cfg4_launches.csv \
   python tools/cfg_steps.py cfg4 --steps 3 --sweeps 1 --resort > $o/cfg4_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_momentum_ordered|k_deformation_rate_ordered" -s 2 -c 2 -o $o/cfg4_tl \
   python tools/cfg_steps.py cfg4 --steps 2 --sweeps 0 > $o/cfg4_tl_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_fast -s 30 -c 1 -o $o/cfg4_sweep \
   python tools/cfg_steps.py cfg4 --steps 0 --sweeps 1 > $o/cfg4_sweep_ncu.log 2>&1
ls -la $o
