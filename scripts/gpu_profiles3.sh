set -x
O=gpurun_out/prof
mkdir -p $O
export HH_ND_CUT=-1 HH_ND_SPLIT=99
HH_SWEEP_STREAMS=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv --log-file $O/launches_bench_sweep_forced.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch_forced.log 2>&1
echo launch_rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_nd_bwd -s 12 -c 1 -o $O/full_cfg2_k_nd_bwd_leaves python scripts/ncu_target.py cfg2 > $O/ncu_full_cfg2_bwd.log 2>&1
echo bwd rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_nd_fwd -s 0 -c 1 -o $O/full_cfg2_k_nd_fwd_leaves python scripts/ncu_target.py cfg2 > $O/ncu_full_cfg2_fwd.log 2>&1
echo fwd rc=$?
