#!/bin/bash
# A/B of the TL-SPH passes: default build vs variant(s) named on the command line (cfg4, cfg3 elastic).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
o=gpurun_out/abtl; mkdir -p $o
for rep in 1 2; do
for lib in default "$@"; do
  if [ $lib = default ]; then unset TLSPH_CUDA_LIB; else export TLSPH_CUDA_LIB=$PWD/paper_2103_08932_b200/lib/libtlsph_cuda_$lib.so; fi
  echo "== $lib" >> $o/ab.log
  timeout 200 python tools/cfg_steps.py cfg4 --steps 12 --sweeps 0 >> $o/ab.log 2>&1
  timeout 200 python tools/cfg_steps.py cfg3 --steps 50 --sweeps 0 >> $o/ab.log 2>&1
done
done
