#!/bin/bash
# A/B/C..: LIBS="A B C" (B = working-tree libhh.so, X = libhh_X.so), sweep bench alternated REPS times;
# then TESTS (pytest -m gpu) on the working-tree library
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${AB_OUT:-ab}; mkdir -p $O
summ() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']['phases']
print(round(d['value']/1e9,4), round(d['ms_per_step'],2), {k:(round(v['avg_us'],1), round(v['frac'],3)) for k,v in r.items()})"; }
for rep in $(seq ${REPS:-3}); do for l in ${LIBS:-A B}; do
  if [ $l = B ]; then unset HH_LIB; else export HH_LIB=$PWD/paper_2104_01439_b200/libhh_$l.so; fi
  echo "$l ${WL:-sweep} $(timeout 300 python bench.py --workload ${WL:-sweep} --no-cpu-baseline --no-cold 2>>$O/err.log | summ)" >> $O/ab.txt
done; done
unset HH_LIB
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest -m gpu -q -x -p no:cacheprovider $TESTS > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
fi
