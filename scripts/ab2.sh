# A/B of cfg2 per-phase times and the sweep: libhh_A.so (baseline) vs libhh.so
for l in A B A B; do
  if [ $l = A ]; then export HH_LIB=$PWD/paper_2104_01439_b200/libhh_A.so; else unset HH_LIB; fi
  echo "$l cfg2 $(python bench.py --workload cfg2 --no-cpu-baseline --steps 2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']['phases']
print(round(d['ms_per_step'],1), {k:(round(v['avg_us'],1)) for k,v in r.items()})")"
  echo "$l $(python scripts/probe_sweep.py 2>&1 | tail -1)"
done
