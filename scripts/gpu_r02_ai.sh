#!/bin/bash
# ncu launch list of the bench's timed step (one engine stream: ncu aborts multi-threaded graph capture), cfg3 too
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ai
mkdir -p $O
timeout 1500 env HH_SWEEP_STREAMS=1 HH_BENCH_PROFILE=1 HH_BENCH_NO_CLOCKS=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 400000 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cold > $O/ncu_bench.log 2>&1; echo "sweep=$?" >> $O/status.txt
timeout 600 env HH_BENCH_PROFILE=1 HH_BENCH_NO_CLOCKS=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv \
  python bench.py --workload cfg3 --steps 1 --warmup 1 --no-cpu-baseline --no-cold > $O/ncu_cfg3.log 2>&1; echo "cfg3=$?" >> $O/status.txt
gzip -f $O/*.csv
