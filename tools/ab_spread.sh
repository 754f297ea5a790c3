#!/bin/bash
# Same-box A/B of the bank-spread FAST sweep rows (TLSPH_SWEEP_SPREAD): sweep times per body.
#   make -C paper_2103_08932_b200/csrc variant V=nospread DEFS=-DTLSPH_SWEEP_SPREAD=0
mkdir -p gpurun_out
for i in 1 2; do
  for L in libtlsph_cuda.so libtlsph_cuda_nospread.so; do
    echo "== $L"
    TLSPH_CUDA_LIB=$PWD/paper_2103_08932_b200/lib/$L python tools/sweep_sizes.py ${CFGS:-cfg2 cfg3 cfg4 cfg5_weak} --sweeps 10
  done
done
