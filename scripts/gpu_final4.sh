# End-of-round measurements (after the factorisation update work)
O=gpurun_out/final4
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_sweep.json 2> $O/bench_sweep.err; echo sweep=$?
timeout 400 python bench.py --workload cfg2 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo cfg2=$?
timeout 400 python bench.py --workload cfg3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo cfg3=$?
timeout 400 python bench.py --workload search --no-cpu-baseline > $O/bench_search.json 2> $O/bench_search.err; echo search=$?
timeout 300 env HH_PROFILE_SETUP=2 python scripts/probe_cfg3.py cfg3 > $O/factor_levels_cfg3.txt 2>&1
timeout 600 env HH_ND_CUT=-1 HH_ND_SPLIT=99 ncu --set full --clock-control none --import-source on -k regex:k_nd_upd -s 300 -c 1 -o $O/full_cfg3_k_nd_upd python scripts/ncu_factor.py cfg3 > /dev/null 2>&1; echo ncu_upd=$?
timeout 900 env HH_BENCH_NO_CLOCKS=1 HH_ND_CUT=-1 HH_ND_SPLIT=99 HH_SWEEP_STREAMS=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $O/launches_bench_sweep.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 1200 python bench.py --workload cfg4 --no-cpu-baseline --steps 2 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo cfg4=$?
timeout 300 python scripts/bench_lfa.py > $O/bench_lfa.json 2> $O/bench_lfa.err; echo lfa=$?
