#!/bin/bash
# session 6: programmatic dependent launch inside the FD chain (HH_FD_PDL=1) A/B: A = off, B = on
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02s6f; mkdir -p $O
summ() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']['phases']
print(round(d['value']/1e9,4), round(d['ms_per_step'],2), round(d['e2e']['value']/1e9,4), {k:(round(v['avg_us'],1), round(v['frac'],3)) for k,v in r.items()})"; }
HH_FD_PDL=1 timeout 600 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_fd.py > $O/pytest_fd_pdl.log 2>&1; echo "fd_tests_pdl=$?" >> $O/status.txt
for n in 534 400 134 34; do
  for l in A B; do
    if [ $l = B ]; then export HH_FD_PDL=1; else unset HH_FD_PDL; fi
    echo "$l probe_fd $n: $(timeout 300 python scripts/probe_fd.py $n 2>&1 | tail -n 1)" >> $O/probe.txt
  done
done
for l in A B A B A B; do
  if [ $l = B ]; then export HH_FD_PDL=1; else unset HH_FD_PDL; fi
  echo "$l sweep $(timeout 300 python bench.py --no-cpu-baseline --no-cold 2>>$O/err.log | summ)" >> $O/ab.txt
done
for l in A B; do
  if [ $l = B ]; then export HH_FD_PDL=1; else unset HH_FD_PDL; fi
  echo "$l cfg3 $(timeout 300 python bench.py --workload cfg3 --no-cpu-baseline --no-cold 2>>$O/err.log | summ)" >> $O/ab.txt
done
export HH_FD_PDL=1
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_goldens.py tests/test_gpu_parity.py > $O/pytest_pdl2.log 2>&1; echo "tests_pdl2=$?" >> $O/status.txt
