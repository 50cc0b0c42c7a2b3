#!/bin/bash
# FD GEMM K-chunk 32 vs 16 per pipeline stage
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02as
mkdir -p $O
HH_LIB=$PWD/paper_2104_01439_b200/libhh_bk32.so timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_fd.py > $O/pytest_bk32.log 2>&1; echo "par=$?" >> $O/status.txt
timeout 400 python scripts/probe_fd.py 134 268 400 534 > $O/probe_bk16.txt 2>&1
HH_LIB=$PWD/paper_2104_01439_b200/libhh_bk32.so timeout 400 python scripts/probe_fd.py 134 268 400 534 > $O/probe_bk32.txt 2>&1
timeout 400 python bench.py --workload cfg3 --no-cpu-baseline --no-cold --steps 5 --warmup 3 > $O/cfg3_bk16.json 2>/dev/null
HH_LIB=$PWD/paper_2104_01439_b200/libhh_bk32.so timeout 400 python bench.py --workload cfg3 --no-cpu-baseline --no-cold --steps 5 --warmup 3 > $O/cfg3_bk32.json 2>/dev/null
