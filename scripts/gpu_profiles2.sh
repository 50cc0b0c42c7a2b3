set -x
O=gpurun_out/prof
mkdir -p $O
export HH_SWEEP_STREAMS=1
ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv --log-file $O/launches_bench_sweep.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo launch_rc=$?
for k in k_nd_bwd k_nd_fwd k_mdot k_update k_pre2d k_post2d; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 3000 -c 1 -o $O/full_sweep_$k python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_$k.log 2>&1
  echo $k rc=$?
done
