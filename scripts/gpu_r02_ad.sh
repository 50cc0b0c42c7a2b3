#!/bin/bash
# ncu --set full of the Krylov kernels and the fused smoothers at the sweep's largest batch (n = 534, B = 8)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ad
mkdir -p $O
for k in k_mdot k_update k_pre2d k_post2d k_fd_gemm; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 300 -c 2 -o $O/$k \
    python scripts/probe_fd.py 534 > $O/ncu_$k.log 2>&1; echo "$k=$?" >> $O/status.txt
done
