#!/bin/bash
# round 2: sweep ND schedule under concurrency: throughput-tuned (default) vs
# latency-tuned (HH_ND_TUNE_CONC=0) vs forced schedules
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02f
mkdir -p $O
run() {  # name, env...
  local name=$1; shift
  timeout 600 env "$@" python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-cold > $O/sweep_$name.json 2> $O/sweep_$name.err
  echo "$name rc=$?" >> $O/status.txt
}
run tuneconc HH_DEBUG=0
run tuneiso HH_ND_TUNE_CONC=0
run perlevel HH_ND_CUT=-1 HH_ND_SPLIT=99
run sub2 HH_ND_CUT=2 HH_ND_SPLIT=99
run tuneconc2 HH_DEBUG=0
