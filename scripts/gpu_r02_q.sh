#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02q
mkdir -p $O
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_bench scripts/cuda/dmma_bench.cu > $O/build.log 2>&1
/tmp/dmma_bench > $O/dmma.json 2>&1; echo "dmma=$?" >> $O/status.txt
timeout 600 env HH_PROFILE_SETUP=2 python scripts/probe_cfg3.py cfg3 > $O/factor_levels_cfg3.txt 2>&1; echo "prof=$?" >> $O/status.txt
