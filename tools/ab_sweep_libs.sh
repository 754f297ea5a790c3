#!/bin/bash
# Same-box A/B of sweep variants: LIBS="a b c" (names under paper_2103_08932_b200/lib, without the
# libtlsph_cuda prefix; "main" = libtlsph_cuda.so), CFGS="cfg2 cfg3 cfg4 cfg5_weak".
for i in 1 2; do
  for L in ${LIBS:-main}; do
    lib=libtlsph_cuda_$L.so; [ "$L" = main ] && lib=libtlsph_cuda.so
    echo "== $lib"
    TLSPH_CUDA_LIB=$PWD/paper_2103_08932_b200/lib/$lib python tools/sweep_sizes.py ${CFGS:-cfg2 cfg3 cfg4 cfg5_weak} --sweeps 10
  done
done
