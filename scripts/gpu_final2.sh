# End-of-round measurements (session 3): tests, bench lines, launch lists, ncu captures
O=gpurun_out/final2
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_sweep.json 2> $O/bench_sweep.err; echo sweep=$?
timeout 400 python bench.py --workload cfg2 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo cfg2=$?
timeout 400 python bench.py --workload cfg3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo cfg3=$?
timeout 400 python bench.py --workload search --no-cpu-baseline > $O/bench_search.json 2> $O/bench_search.err; echo search=$?
timeout 300 python scripts/bench_lfa.py > $O/bench_lfa.json 2> $O/bench_lfa.err; echo lfa=$?
timeout 300 env HH_ND_LEVEL_TIMING=1 python scripts/probe_nd_levels.py cfg2 > $O/nd_levels_cfg2.txt 2>&1
timeout 900 env HH_BENCH_NO_CLOCKS=1 HH_ND_CUT=-1 HH_ND_SPLIT=99 HH_SWEEP_STREAMS=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $O/launches_bench_sweep.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file $O/launches_cfg2.csv python scripts/ncu_target.py cfg2 > $O/ncu_cfg2.log 2>&1; echo ncu_cfg2=$?
for k in k_pre2d k_post2d k_mdot k_update k_nd_flow_bwd k_nd_flow_fwd; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 1 -o $O/full_cfg2_$k python scripts/ncu_target.py cfg2 > $O/ncu_full_$k.log 2>&1; echo full_$k=$?
done
timeout 900 python bench.py --workload cfg4 --no-cpu-baseline --steps 2 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo cfg4=$?
