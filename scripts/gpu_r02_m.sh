#!/bin/bash
# round 2: sweep with larger ND leaves (fewer dependent levels per coarse solve)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02m
mkdir -p $O
run() {
  local name=$1; shift
  timeout 600 env "$@" python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-cold > $O/sweep_$name.json 2> $O/sweep_$name.err
  echo "$name rc=$?" >> $O/status.txt
}
run leaf64 HH_ND_LEAF=64
run leaf128 HH_ND_LEAF=128
run leaf256 HH_ND_LEAF=256
run leaf32 HH_ND_LEAF=32
