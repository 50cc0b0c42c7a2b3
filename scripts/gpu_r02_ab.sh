#!/bin/bash
# sweep engine streams 1..3 (x node budget) with the FD coarse solve
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ab
mkdir -p $O
for st in 1 2 3; do for nb in 2.4e6 9.6e6 4e7; do
  timeout 300 env HH_SWEEP_STREAMS=$st HH_SWEEP_NODES=$nb python bench.py --no-cpu-baseline --no-cold --steps 2 --warmup 2 > $O/sweep_st${st}_nb${nb}.json 2>/dev/null; echo "st$st nb$nb=$?" >> $O/status.txt
done; done
