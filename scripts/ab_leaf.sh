# ND leaf size: cfg2 phases, sweep wall, sweep setup share
for leaf in 64 32 16; do
  export HH_ND_LEAF=$leaf
  echo "leaf=$leaf cfg2 $(python bench.py --workload cfg2 --no-cpu-baseline --steps 2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']['phases']
print(round(d['ms_per_step'],1), {k:(round(v['avg_us'],1)) for k,v in r.items()})")"
  echo "leaf=$leaf $(python scripts/probe_sweep.py 2>&1 | tail -1)"
  echo "leaf=$leaf $(python scripts/probe_sweep_split.py 2>&1 | tr '\n' ' ')"
done
