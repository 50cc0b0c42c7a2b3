#!/bin/bash
# A/B (sweep only, 3 alternations) + per-n-group probe of the working tree
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${AB_OUT:-ab}; mkdir -p $O
summ() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']['phases']
print(round(d['value']/1e9,4), round(d['ms_per_step'],2), {k:(round(v['avg_us'],1), round(v['frac'],3)) for k,v in r.items()})"; }
for l in A B A B A B; do
  if [ $l = A ]; then export HH_LIB=$PWD/paper_2104_01439_b200/libhh_A.so; else unset HH_LIB; fi
  echo "$l sweep $(timeout 300 python bench.py --no-cpu-baseline --no-cold 2>>$O/err.log | summ)" >> $O/ab.txt
done
unset HH_LIB
timeout 600 python scripts/probe_groups_full.py > $O/groups.txt 2>&1
