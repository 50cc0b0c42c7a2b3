#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02s
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $O/launches_cfg3_setup.csv python scripts/probe_cfg3.py cfg3 > $O/ncu.log 2>&1; echo "ncu=$?" >> $O/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_nd_upd_mma" -s 3000 -c 1 -o $O/full_upd_mma_cfg3 python scripts/probe_cfg3.py cfg3 > $O/ncu2.log 2>&1; echo "ncu2=$?" >> $O/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_nd_piv" -s 3000 -c 1 -o $O/full_piv_cfg3 python scripts/probe_cfg3.py cfg3 > $O/ncu3.log 2>&1; echo "ncu3=$?" >> $O/status.txt
