#!/bin/bash
# locate the crash under ncu: python faulthandler; ND vs FD sweep; single-problem bench
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ah
mkdir -p $O
N="ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv"
timeout 600 env HH_BENCH_NO_CLOCKS=1 $N --log-file $O/l_fd.csv python -X faulthandler bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cold > $O/fd.log 2>&1; echo "fd=$?" >> $O/status.txt
timeout 600 env HH_BENCH_NO_CLOCKS=1 $N --log-file $O/l_nd.csv python -X faulthandler bench.py --coarse-solver nd --steps 1 --warmup 1 --no-cpu-baseline --no-cold > $O/nd.log 2>&1; echo "nd=$?" >> $O/status.txt
timeout 600 env HH_BENCH_NO_CLOCKS=1 $N --log-file $O/l_cfg3.csv python -X faulthandler bench.py --workload cfg3 --steps 1 --warmup 1 --no-cpu-baseline --no-cold > $O/cfg3.log 2>&1; echo "cfg3=$?" >> $O/status.txt
timeout 600 env HH_BENCH_NO_CLOCKS=1 HH_SWEEP_STREAMS=1 $N --log-file $O/l_fd1.csv python -X faulthandler scripts/traffic_target.py sweep /tmp/t.json > $O/tt.log 2>&1; echo "tt=$?" >> $O/status.txt
gzip -f $O/*.csv
