#!/bin/bash
# full -m gpu suite + smoke + default bench (cpu_baseline, cold e2e) + ncu launch list of the bench command
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ae
mkdir -p $O
timeout 2400 python -m pytest -q -p no:cacheprovider -m gpu tests --durations=20 > $O/pytest_gpu.log 2>&1; echo "gpu=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/status.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench=$?" >> $O/status.txt
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref=$?" >> $O/status.txt
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 80000 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cold > $O/ncu_bench.log 2>&1; echo "ncu_launch=$?" >> $O/status.txt
gzip -f $O/launches_bench.csv
