#!/bin/bash
# ncu --set full of one streamed sweep phase on the cfg5-weak body (run on the GPU box, one GPU).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
out=${1:-gpurun_out/sweep_scale}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_fast -s 60 -c 1 -o "$out" \
  python tools/sweep_sizes.py cfg5_weak --sweeps 1
