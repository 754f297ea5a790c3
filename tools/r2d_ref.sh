#!/bin/bash
# Round-2d: the reference arm (oracle alone) as the driver launches it, and the N = 2 protocol
# run of the sharded cfg5 loop on one device (TLSPH_BENCH_ONE_DEVICE=1: two ranks share GPU 0).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
o=gpurun_out/r2d; mkdir -p $o
( time timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $o/bench_reference.json 2> $o/bench_reference.err ) 2> $o/bench_reference.time; echo "ref rc=$?"
tail -c 600 $o/bench_reference.json; cat $o/bench_reference.time
( time TLSPH_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 5 --warmup 3 --scale-layers 60 > $o/bench_n2_onedev.json 2> $o/bench_n2_onedev.err ) 2> $o/bench_n2.time; echo "n2 rc=$?"
tail -c 1500 $o/bench_n2_onedev.json; tail -5 $o/bench_n2_onedev.err; cat $o/bench_n2.time
