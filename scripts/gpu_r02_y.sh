#!/bin/bash
# round 2 (session 4): FD slots + warp-parallel roots + tile choice: parity + tile A/B
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02y
mkdir -p $O
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_fd.py tests/test_gpu_parity.py > $O/pytest.log 2>&1; echo "par=$?" >> $O/status.txt
for t in 0 32 48 64; do
  timeout 600 env HH_FD_TILE=$t python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/bench_sweep_t$t.json 2> $O/bench_sweep_t$t.err; echo "sweep_$t=$?" >> $O/status.txt
  timeout 600 env HH_FD_TILE=$t python bench.py --workload cfg3 --no-cpu-baseline --no-cold --steps 5 --warmup 3 > $O/bench_cfg3_t$t.json 2> $O/bench_cfg3_t$t.err; echo "cfg3_$t=$?" >> $O/status.txt
done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/traffic_sweep.csv \
  python scripts/traffic_target.py sweep $O/traffic_sweep_timers.json > $O/traffic_sweep.log 2>&1; echo "traffic_sweep=$?" >> $O/status.txt
gzip -f $O/traffic_sweep.csv
