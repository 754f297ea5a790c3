#!/bin/bash
# Round-2c GPU pass: parity suite, staged/streamed choice for cfg3 with bank-spread rows, ncu --set
# full of one streamed cfg4 sweep phase (bank-spread rows) next to the slot-order variant library.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
o=gpurun_out/r2c; mkdir -p $o
python -m pytest tests -m gpu -q > $o/gputest.log 2>&1; echo "rc=$?" >> $o/gputest.log; tail -15 $o/gputest.log | cut -c1-180
for st in 0 1; do TLSPH_SWEEP_STREAM=$st python tools/sweep_sizes.py cfg2 cfg3 --sweeps 20; done 2>&1 | tee $o/cfg3_stream_ab.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_fast -s 30 -c 1 -o $o/cfg4_sweep_spread \
   python tools/cfg_steps.py cfg4 --steps 0 --sweeps 1 > $o/cfg4_sweep_ncu.log 2>&1
ls -la $o
