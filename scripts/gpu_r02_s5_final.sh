#!/bin/bash
# final evidence pass (session 5): full -m gpu suite, smoke, default bench + reference arm, traffic (sweep, cfg3),
# ncu launch lists of the timed steps, ncu --set full of the dominant kernels
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02s5
mkdir -p $O
timeout 2400 python -m pytest -q -p no:cacheprovider -m gpu tests --durations=15 > $O/pytest_gpu.log 2>&1; echo "gpu=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/status.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench=$?" >> $O/status.txt
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref=$?" >> $O/status.txt
for w in cfg0 cfg2 cfg3; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-cold > $O/bench_$w.json 2> $O/bench_$w.err; echo "$w=$?" >> $O/status.txt
done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 900 env HH_BENCH_NO_CLOCKS=1 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/traffic_sweep.csv \
  python scripts/traffic_target.py sweep $O/traffic_sweep_timers.json > $O/traffic_sweep.log 2>&1; echo "traffic_sweep=$?" >> $O/status.txt
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/traffic_cfg2.csv \
  python scripts/traffic_target.py cfg2 $O/traffic_cfg2_timers.json > $O/traffic_cfg2.log 2>&1; echo "traffic_cfg2=$?" >> $O/status.txt
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/traffic_cfg3.csv \
  python scripts/traffic_target.py cfg3 $O/traffic_cfg3_timers.json > $O/traffic_cfg3.log 2>&1; echo "traffic_cfg3=$?" >> $O/status.txt
timeout 1500 env HH_SWEEP_STREAMS=1 HH_BENCH_PROFILE=1 HH_BENCH_NO_CLOCKS=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 400000 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cold > $O/ncu_bench.log 2>&1; echo "launch=$?" >> $O/status.txt
for k in k_mdot k_update k_fd_gemm; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 300 -c 1 -o $O/full_$k \
    python scripts/probe_fd.py 534 > $O/ncu_full_$k.log 2>&1; echo "full_$k=$?" >> $O/status.txt
done
gzip -f $O/*.csv
