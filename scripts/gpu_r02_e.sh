#!/bin/bash
# round 2: register-carry z-marching 3D kernels + per-rank packed-S placement of the distributed coarse solve
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02e
mkdir -p $O
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_dist_coarse.py tests/test_gpu_nd_forced.py tests/test_gpu_fullsize.py > $O/pytest_3d.log 2>&1; echo "par3d=$?" >> $O/status.txt
timeout 900 python bench.py --workload cfg3 --no-cpu-baseline --no-cold --steps 2 --warmup 2 > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo "cfg3=$?" >> $O/status.txt
timeout 1500 python bench.py --workload cfg4 --no-cpu-baseline --no-cold --steps 1 --warmup 1 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "cfg4=$?" >> $O/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_march3d -s 6 -c 2 -o $O/full_march3d_cfg4 python scripts/ncu_target.py cfg4 > $O/ncu_march.log 2>&1; echo "ncu_march=$?" >> $O/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_march3d -s 6 -c 2 -o $O/full_march3d_cfg3 python scripts/ncu_target.py cfg3 > $O/ncu_march3.log 2>&1; echo "ncu_march3=$?" >> $O/status.txt
