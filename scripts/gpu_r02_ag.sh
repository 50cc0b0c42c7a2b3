#!/bin/bash
# ncu launch list of the bench command without the in-process NVML clock sampler
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ag
mkdir -p $O
timeout 900 env HH_BENCH_NO_CLOCKS=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 80000 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cold > $O/ncu_bench.log 2>&1; echo "noclk=$?" >> $O/status.txt
gzip -f $O/*.csv
