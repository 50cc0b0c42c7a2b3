#!/bin/bash
# column strips with a one-row-ahead load: post (default lib) and pre too (libhh_pre1.so)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ap
mkdir -p $O
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_slabs.py > $O/pytest.log 2>&1; echo "par=$?" >> $O/status.txt
HH_LIB=$PWD/paper_2104_01439_b200/libhh_pre1.so timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py > $O/pytest_pre1.log 2>&1; echo "par1=$?" >> $O/status.txt
timeout 400 python scripts/probe_fd.py 68 268 534 > $O/probe_post.txt 2>&1
HH_LIB=$PWD/paper_2104_01439_b200/libhh_pre1.so timeout 400 python scripts/probe_fd.py 68 268 534 > $O/probe_pre1.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/sweep_post.json 2>/dev/null; echo "s=$?" >> $O/status.txt
HH_LIB=$PWD/paper_2104_01439_b200/libhh_pre1.so timeout 600 python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/sweep_pre1.json 2>/dev/null; echo "s1=$?" >> $O/status.txt
