#!/bin/bash
# session 6: A/B of HH_SWEEP_FD_WAVE (FD batches sized to whole waves of the GEMM tiles): A = off, B = on
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02s6d; mkdir -p $O
summ() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']['phases']
print(round(d['value']/1e9,4), round(d['ms_per_step'],2), round(d['e2e']['value']/1e9,4), {k:(round(v['avg_us'],1), round(v['frac'],3), v['launches']) for k,v in r.items()})"; }
for l in A B A B A B; do
  if [ $l = B ]; then export HH_SWEEP_FD_WAVE=1; else unset HH_SWEEP_FD_WAVE; fi
  echo "$l sweep $(timeout 300 python bench.py --no-cpu-baseline --no-cold 2>>$O/err.log | summ)" >> $O/ab.txt
done
export HH_SWEEP_FD_WAVE=1
timeout 600 python scripts/probe_groups_full.py > $O/groups_wave.txt 2>&1
timeout 600 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_goldens.py tests/test_gpu_sweep_share.py -k "cfg1 or sweep" > $O/pytest_wave.log 2>&1; echo "tests_wave=$?" >> $O/status.txt
