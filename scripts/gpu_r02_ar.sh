#!/bin/bash
# lockstep waste: max batch size x engine streams
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ar
mkdir -p $O
for mb in 256 32 16; do for st in 3 6; do
  timeout 300 env HH_SWEEP_MAX_BATCH=$mb HH_SWEEP_STREAMS=$st python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 2 > $O/sweep_mb${mb}_st${st}.json 2>/dev/null; echo "mb$mb st$st=$?" >> $O/status.txt
done; done
