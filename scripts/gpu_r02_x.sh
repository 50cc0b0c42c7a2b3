#!/bin/bash
# round 2 (session 4): FD coarse solve -- parity, bench lines, ncu traffic + launch list + full capture of k_fd_gemm
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02x
mkdir -p $O
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fd.py > $O/pytest.log 2>&1; echo "par=$?" >> $O/status.txt
timeout 600 python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/bench_sweep.json 2> $O/bench_sweep.err; echo "sweep=$?" >> $O/status.txt
timeout 600 python bench.py --workload cfg3 --no-cpu-baseline --no-cold --steps 5 --warmup 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo "cfg3=$?" >> $O/status.txt
timeout 600 python bench.py --workload cfg0 --no-cpu-baseline --no-cold --steps 5 --warmup 3 > $O/bench_cfg0.json 2> $O/bench_cfg0.err; echo "cfg0=$?" >> $O/status.txt
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/traffic_sweep.csv \
  python scripts/traffic_target.py sweep $O/traffic_sweep_timers.json > $O/traffic_sweep.log 2>&1; echo "traffic_sweep=$?" >> $O/status.txt
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/traffic_cfg3.csv \
  python scripts/traffic_target.py cfg3 $O/traffic_cfg3_timers.json > $O/traffic_cfg3.log 2>&1; echo "traffic_cfg3=$?" >> $O/status.txt
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_fd_gemm -s 400 -c 4 \
  -o $O/fd_gemm python scripts/traffic_target.py sweep /tmp/t.json > $O/ncu_full.log 2>&1; echo "ncu_full=$?" >> $O/status.txt
gzip -f $O/traffic_sweep.csv $O/traffic_cfg3.csv
