#!/bin/bash
# A/B: slots loaded ahead per thread in the slot-order TL-SPH passes (TLSPH_TL_OU variants).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
o=gpurun_out/abou; mkdir -p $o
for lib in default ou2 ou3 ou4 default ou2; do
  if [ $lib = default ]; then unset TLSPH_CUDA_LIB; else export TLSPH_CUDA_LIB=$PWD/paper_2103_08932_b200/lib/libtlsph_cuda_$lib.so; fi
  echo "== $lib" >> $o/ab.log
  timeout 200 python tools/cfg_steps.py cfg4 --steps 12 --sweeps 0 >> $o/ab.log 2>&1
  timeout 200 python tools/cfg_steps.py cfg3 --steps 50 --sweeps 0 >> $o/ab.log 2>&1
done
