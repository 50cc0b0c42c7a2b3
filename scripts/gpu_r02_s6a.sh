#!/bin/bash
# session 6: FD GEMM 3-stage cp.async pipeline (48 x 48 tiles) A/B: A = libhh_A.so (FD_ST48=2), B = working tree (3);
# FD parity subset first, then the sweep A/B and the per-size FD probe of both
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02s6a; mkdir -p $O
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_fd.py tests/test_gpu_goldens.py > $O/pytest_fd.log 2>&1; echo "fd_tests=$?" >> $O/status.txt
for n in 534 268 468; do
  for l in A B; do
    if [ $l = A ]; then export HH_LIB=$PWD/paper_2104_01439_b200/libhh_A.so; else unset HH_LIB; fi
    echo "$l probe_fd $n: $(timeout 300 python scripts/probe_fd.py $n 2>&1 | tail -n 3 | tr '\n' ' ')" >> $O/probe.txt
  done
done
unset HH_LIB
AB_OUT=r02s6a bash scripts/ab_s5b.sh
for l in A B; do
  if [ $l = A ]; then export HH_LIB=$PWD/paper_2104_01439_b200/libhh_A.so; else unset HH_LIB; fi
  timeout 300 python bench.py --workload cfg3 --no-cpu-baseline --no-cold > $O/bench_cfg3_$l.json 2>> $O/err.log
done
