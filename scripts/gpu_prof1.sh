set -x
HH_PROFILE_SETUP=1 python scripts/probe_setup2.py cfg2 cfg3 > gpurun_out/probe_setup_b.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_cfg2.csv python scripts/ncu_target.py cfg2 > gpurun_out/ncu_l.log 2>&1
for k in k_mdot k_update k_nd_bwd k_nd_fwd k_pre2d k_post2d; do
ncu --set full --clock-control none --import-source on -k regex:$k -s 150 -c 1 -o gpurun_out/full_$k python scripts/ncu_target.py cfg2 > gpurun_out/ncu_$k.log 2>&1
done
