# A/B of library variants on the cfg3 elastic step: LIBS="libtlsph_cuda.so libtlsph_cuda_x.so" bash tools/ab_cfg3.sh
for i in 1 2; do for L in $LIBS; do echo -n "$L "; TLSPH_CUDA_LIB=paper_2103_08932_b200/lib/$L python tools/cfg3_step.py ${STEPS:-100} | tail -1; done; done
