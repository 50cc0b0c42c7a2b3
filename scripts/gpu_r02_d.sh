#!/bin/bash
# round 2: sweep batching A/B (node budget per batch x engine streams), launch list
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02d
mkdir -p $O
for NB in 1.2e6 2.4e6 4.8e6; do
  for ST in 8 12; do
    timeout 600 env HH_SWEEP_NODES=$NB HH_SWEEP_STREAMS=$ST python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-cold \
      > $O/sweep_nb${NB}_st${ST}.json 2> $O/sweep_nb${NB}_st${ST}.err
    echo "nb=$NB st=$ST rc=$?" >> $O/status.txt
  done
done
timeout 1800 env HH_SWEEP_STREAMS=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv \
  --log-file $O/launches_bench_1stream.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cold \
  > $O/ncu_bench.log 2>&1; echo "ncu_launch=$?" >> $O/status.txt
gzip -f $O/launches_bench_1stream.csv
