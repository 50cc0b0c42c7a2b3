#!/bin/bash
# FD tile 48 probe + sweep stream / batch-size A/B with the FD coarse solve
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02aa
mkdir -p $O
HH_FD_TILE=48 timeout 400 python scripts/probe_fd.py > $O/probe_fd_t48.txt 2>&1
for st in 4 8 12; do for nb in 2.4e6 4.8e6 9.6e6; do
  timeout 300 env HH_SWEEP_STREAMS=$st HH_SWEEP_NODES=$nb python bench.py --no-cpu-baseline --no-cold --steps 2 --warmup 2 > $O/sweep_st${st}_nb${nb}.json 2>/dev/null; echo "st$st nb$nb=$?" >> $O/status.txt
done; done
