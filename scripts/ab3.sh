for l in A B A B; do
  if [ $l = A ]; then export HH_LIB=$PWD/paper_2104_01439_b200/libhh_A.so; else unset HH_LIB; fi
  echo "$l cfg2 $(python bench.py --workload cfg2 --no-cpu-baseline --steps 2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']['phases']
print(round(d['ms_per_step'],1), {k:(round(v['avg_us'],1)) for k,v in r.items()})")"
done
for l in A B; do
  if [ $l = A ]; then export HH_LIB=$PWD/paper_2104_01439_b200/libhh_A.so; else unset HH_LIB; fi
  echo "$l cfg4 $(HH_TIMING=1 python -c "
import sys, time, torch
sys.path.insert(0, '.')
import paper_2104_01439_b200.hh as hh
from workloads import config_spec
spec = config_spec('cfg4')
gp = hh.Problem.from_spec(spec)
b = torch.from_numpy(spec.rhs()).cuda()
gp.fgmres_solve(b, o=hh.opts(restart=50, rtol=1e-6))
gp.reset_timers(True)
x, r = gp.fgmres_solve(b, o=hh.opts(restart=50, rtol=1e-6))
t = gp.read_timers()
print(r['iterations'], {p: round(1e3 * t[p]['ms'] / max(t[p]['launches'], 1), 1) for p in hh.PHASES})
" 2>&1 | tail -1)"
done
