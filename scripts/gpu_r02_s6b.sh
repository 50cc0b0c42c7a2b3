#!/bin/bash
# session 6: FD GEMM K-chunk 12 (A stage stride 12, no padding) with 3 stages (C) or 2 stages (D) vs the default (16-k chunks, 2 stages)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02s6b; mkdir -p $O
for n in 500 268 400 534 134; do
  for l in base C D; do
    if [ $l = base ]; then unset HH_LIB; else export HH_LIB=$PWD/paper_2104_01439_b200/libhh_$l.so; fi
    echo "$l probe_fd $n: $(timeout 300 python scripts/probe_fd.py $n 2>&1 | tail -n 1)" >> $O/probe.txt
  done
done
export HH_LIB=$PWD/paper_2104_01439_b200/libhh_C.so
timeout 600 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_fd.py > $O/pytest_fd_C.log 2>&1; echo "fd_tests_C=$?" >> $O/status.txt
