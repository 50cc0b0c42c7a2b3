export HH_ND_CUT=1 HH_ND_SPLIT=12
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches_cfg2_forced.csv python scripts/ncu_target.py cfg2 > gpurun_out/ncu_l2.log 2>&1
for k in k_mdot k_update k_pre2d k_post2d; do
ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 1 -o gpurun_out/full_$k python scripts/ncu_target.py cfg2 > gpurun_out/ncu_$k.log 2>&1
done
