#!/bin/bash
# round 2: evidence pass (smoke, FP64 peak, sanitizer on the dataflow ND kernels,
# ncu DRAM traffic per phase, ncu launch list of the bench command)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02b
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/status.txt
timeout 120 python -c "
import paper_2104_01439_b200.hh as hh, json
t, mhz = hh.fp64_peak()
print(json.dumps({'fp64_tflops': t, 'nominal_sm_mhz': mhz}))" > $O/fp64_peak.json 2>&1; echo "peak=$?" >> $O/status.txt
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python scripts/sanitize_flow.py > $O/racecheck_flow.txt 2>&1; echo "racecheck=$?" >> $O/status.txt
timeout 900 compute-sanitizer --tool synccheck python scripts/sanitize_flow.py > $O/synccheck_flow.txt 2>&1; echo "synccheck=$?" >> $O/status.txt
timeout 900 compute-sanitizer --tool memcheck python scripts/sanitize_flow.py > $O/memcheck_flow.txt 2>&1; echo "memcheck=$?" >> $O/status.txt
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 1500 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/traffic_sweep.csv \
  python scripts/traffic_target.py sweep $O/traffic_sweep_timers.json > $O/traffic_sweep.log 2>&1; echo "traffic_sweep=$?" >> $O/status.txt
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/traffic_cfg2.csv \
  python scripts/traffic_target.py cfg2 $O/traffic_cfg2_timers.json > $O/traffic_cfg2.log 2>&1; echo "traffic_cfg2=$?" >> $O/status.txt
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cold > $O/ncu_bench.log 2>&1; echo "ncu_launch=$?" >> $O/status.txt
gzip -f $O/launches_bench.csv $O/traffic_sweep.csv
