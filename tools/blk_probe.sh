o=gpurun_out/blk; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "blocked or tiling" > $o/test.log 2>&1; echo rc=$? >> $o/test.log
for b in 0 auto 24,6 16,4 32,8 12,3 40,10; do
  if [ $b = auto ]; then unset TLSPH_SWEEP_BLOCK; else export TLSPH_SWEEP_BLOCK=$b; fi
  echo "== $b" >> $o/sizes.log
  timeout 600 python tools/sweep_sizes.py cfg4 cfg5_weak --sweeps 5 >> $o/sizes.log 2>&1
done
