#!/bin/bash
# reproduce the ncu launch-list crash: streams 3 / 8 / 1
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02af
mkdir -p $O
for st in 3 8 1; do
timeout 900 env HH_SWEEP_STREAMS=$st ncu --metrics gpu__time_duration.sum --clock-control none -c 80000 --csv --log-file $O/launches_st$st.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cold > $O/ncu_st$st.log 2>&1; echo "st$st=$?" >> $O/status.txt
done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-cold > $O/plain.json 2> $O/plain.err; echo "plain=$?" >> $O/status.txt
gzip -f $O/*.csv
