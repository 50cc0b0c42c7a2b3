#!/bin/bash
# 48-tile occupancy (2 vs 3 CTAs/SM) and tile choice with the 3M product
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ak
mkdir -p $O
for t in 0 32 48; do HH_FD_TILE=$t timeout 400 python scripts/probe_fd.py 134 200 268 400 468 534 > $O/probe_t$t.txt 2>&1; done
timeout 600 python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/bench_sweep.json 2> $O/bench_sweep.err; echo "sweep=$?" >> $O/status.txt
