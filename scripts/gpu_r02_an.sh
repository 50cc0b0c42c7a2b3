#!/bin/bash
# exclusive timed iterations in the concurrent sweep: throughput + phase fractions, on vs off
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02an
mkdir -p $O
for x in 1 0 1 0; do
  timeout 600 env HH_SWEEP_EXCL_TIMING=$x python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/sweep_x$x.json 2> $O/sweep_x$x.err; echo "x$x=$?" >> $O/status.txt
  cat $O/sweep_x$x.json >> $O/all.jsonl
done
timeout 300 env HH_TIMING_EVERY=16 python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/sweep_x1_te16.json 2>/dev/null; echo "te16=$?" >> $O/status.txt
