set -x
O=gpurun_out/final
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
python bench.py > $O/bench_sweep.json 2> $O/bench_sweep.err
python bench.py --workload cfg2 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python bench.py --workload cfg3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python bench.py --workload search --no-cpu-baseline > $O/bench_search.json 2> $O/bench_search.err
timeout 900 python bench.py --workload cfg4 --no-cpu-baseline --steps 2 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
HH_ND_LEVEL_TIMING=1 python scripts/probe_nd_levels.py cfg4 > $O/nd_levels_cfg4.txt 2>&1
HH_ND_LEVEL_TIMING=1 python scripts/probe_nd_levels.py cfg2 > $O/nd_levels_cfg2.txt 2>&1
HH_BENCH_NO_CLOCKS=1 HH_ND_CUT=-1 HH_ND_SPLIT=99 HH_SWEEP_STREAMS=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $O/launches_bench_sweep.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo ncu_rc=$?
