#!/bin/bash
# sweep: host status-check interval x engine streams
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ac
mkdir -p $O
for st in 1 3 8; do for ce in 1 4 16; do
  timeout 300 env HH_SWEEP_STREAMS=$st python bench.py --check-every $ce --no-cpu-baseline --no-cold --steps 2 --warmup 2 > $O/sweep_st${st}_ce${ce}.json 2>/dev/null; echo "st$st ce$ce=$?" >> $O/status.txt
done; done
