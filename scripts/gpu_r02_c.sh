#!/bin/bash
# round 2: distributed coarse solve + z-marching 3D kernels: parity, then timing
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02c
mkdir -p $O
timeout 1800 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_dist_coarse.py -k "not fullsize" > $O/pytest_dist.log 2>&1; echo "dist=$?" >> $O/status.txt
timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_nd_forced.py tests/test_gpu_fullsize.py tests/test_gpu_search.py > $O/pytest_3d.log 2>&1; echo "par3d=$?" >> $O/status.txt
timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_goldens.py -k cfg1 > $O/pytest_gold_cfg1.log 2>&1; echo "gold1=$?" >> $O/status.txt
timeout 900 python bench.py --workload cfg3 --no-cpu-baseline --no-cold --steps 2 --warmup 2 > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo "cfg3=$?" >> $O/status.txt
timeout 900 env HH_3D_NAIVE=1 python bench.py --workload cfg3 --no-cpu-baseline --no-cold --steps 2 --warmup 2 > $O/bench_cfg3_naive.json 2> $O/bench_cfg3_naive.err; echo "cfg3n=$?" >> $O/status.txt
timeout 1500 python bench.py --workload cfg4 --no-cpu-baseline --no-cold --steps 1 --warmup 1 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "cfg4=$?" >> $O/status.txt
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_dist_coarse.py -k fullsize > $O/pytest_dist_full.log 2>&1; echo "distfull=$?" >> $O/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_march3d -s 6 -c 2 -o $O/full_march3d_cfg4 python scripts/ncu_target.py cfg4 > $O/ncu_march.log 2>&1; echo "ncu_march=$?" >> $O/status.txt
