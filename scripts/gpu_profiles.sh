# Round-1 profile set (run from the repo root on the GPU box).
set -x
O=gpurun_out/prof
mkdir -p $O
python bench.py > $O/bench_sweep.json 2> $O/bench_sweep.err
python bench.py --workload cfg2 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python bench.py --workload cfg3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python bench.py --workload search --no-cpu-baseline > $O/bench_search.json 2> $O/bench_search.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 25000 --csv --log-file $O/launches_bench_sweep.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv --log-file $O/launches_cfg2.csv python scripts/ncu_target.py cfg2 > /dev/null 2>&1
for k in k_nd_bwd k_nd_fwd k_mdot k_update k_pre2d k_post2d; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 600 -c 1 -o $O/full_sweep_$k python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_$k.log 2>&1
done
