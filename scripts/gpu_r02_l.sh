#!/bin/bash
# round 2: per-kernel DRAM traffic of the 3D single solves (cfg3, cfg4)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02l
mkdir -p $O
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 1200 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/traffic_cfg3.csv \
  python scripts/traffic_target.py cfg3 $O/traffic_cfg3_timers.json > $O/traffic_cfg3.log 2>&1; echo "t3=$?" >> $O/status.txt
timeout 1800 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/traffic_cfg4.csv \
  python scripts/traffic_target.py cfg4 $O/traffic_cfg4_timers.json > $O/traffic_cfg4.log 2>&1; echo "t4=$?" >> $O/status.txt
gzip -f $O/traffic_cfg3.csv $O/traffic_cfg4.csv
