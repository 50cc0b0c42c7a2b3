#!/bin/bash
# session 6 closing pass: FD chain PDL on by default; full -m gpu suite, smoke, default bench + reference arm, cfg2/cfg3 lines,
# ncu launch list of the timed step
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02s6g; mkdir -p $O
timeout 2400 python -m pytest -q -p no:cacheprovider -m gpu tests --durations=8 > $O/pytest_gpu.log 2>&1; echo "gpu=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/status.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench=$?" >> $O/status.txt
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref=$?" >> $O/status.txt
for w in cfg2 cfg3; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-cold > $O/bench_$w.json 2> $O/bench_$w.err; echo "$w=$?" >> $O/status.txt
done
timeout 1500 env HH_SWEEP_STREAMS=1 HH_BENCH_PROFILE=1 HH_BENCH_NO_CLOCKS=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 400000 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cold > $O/ncu_bench.log 2>&1; echo "launch=$?" >> $O/status.txt
gzip -f $O/*.csv
