#!/bin/bash
# session 6: 3D z-chunk count by the rounds x plane-steps cost model (default) vs the old ">= 4 CTAs per SM" rule
# (HH_3D_NZC_OLD=1): cfg3 / cfg4-medium bench lines A/B, 3D fine probe, then the full -m gpu suite + smoke at the new default
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02s6e; mkdir -p $O
summ() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']['phases']
print(round(d['value']/1e9,4), round(d['ms_per_step'],3), {k:(round(v['avg_us'],1), round(v['frac'],3)) for k,v in r.items()})"; }
for l in A B A B; do
  if [ $l = A ]; then export HH_3D_NZC_OLD=1; else unset HH_3D_NZC_OLD; fi
  echo "$l cfg3 $(timeout 300 python bench.py --workload cfg3 --no-cpu-baseline --no-cold 2>>$O/err.log | summ)" >> $O/ab.txt
done
for z in 2 3 4 6; do
  echo "NZC=$z cfg3 $(HH_3D_NZC=$z timeout 300 python bench.py --workload cfg3 --no-cpu-baseline --no-cold 2>>$O/err.log | summ)" >> $O/ab.txt
done
for l in A B; do
  if [ $l = A ]; then export HH_3D_NZC_OLD=1; else unset HH_3D_NZC_OLD; fi
  echo "$l probe_3d cfg3 $(timeout 300 python scripts/probe_3d.py cfg3 2>>$O/err.log | tail -n 1)" >> $O/probe3d.txt
done
unset HH_3D_NZC_OLD
timeout 2400 python -m pytest -q -p no:cacheprovider -m gpu tests --durations=5 > $O/pytest_gpu.log 2>&1; echo "gpu=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/status.txt
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench=$?" >> $O/status.txt
timeout 300 python bench.py --workload cfg3 --no-cpu-baseline --no-cold > $O/bench_cfg3.json 2>> $O/err.log
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline --no-cold > $O/bench_cfg2.json 2>> $O/err.log
for l in A B; do
  if [ $l = A ]; then export HH_3D_NZC_OLD=1; else unset HH_3D_NZC_OLD; fi
  echo "$l probe_3d cfg4 $(timeout 600 python scripts/probe_3d.py cfg4 2>>$O/err.log | tail -n 1)" >> $O/probe3d.txt
done
unset HH_3D_NZC_OLD
