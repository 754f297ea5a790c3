#!/bin/bash
# e2e through the C++ operator API: pinned (tlsph::pin_host_memory) vs pageable caller storage.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
o=gpurun_out/e2e; mkdir -p $o
L=paper_2103_08932_b200/lib/tlsph-operator-loop
for hm in pinned pageable; do
  timeout 300 $L sweep 50 3 fast $hm >> $o/e2e.log 2>&1
  timeout 600 $L loop 10 3 fast $hm >> $o/e2e.log 2>&1
done
