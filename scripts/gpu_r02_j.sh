#!/bin/bash
# round 2: cp.async staging in the z-marching kernels: A/B (2 vs 3 CTAs/SM) + parity + cfg4 phases
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02j
mkdir -p $O
timeout 600 python scripts/probe_3d.py > $O/probe_march.json 2> $O/probe_march.err; echo "m=$?" >> $O/status.txt
timeout 600 env HH_3D_MINB=3 python scripts/probe_3d.py > $O/probe_march3.json 2> $O/probe_march3.err; echo "m3=$?" >> $O/status.txt
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_nd_forced.py tests/test_gpu_fullsize.py tests/test_gpu_dist_coarse.py -k "not fullsize or cfg2" > $O/pytest_3d.log 2>&1; echo "par=$?" >> $O/status.txt
timeout 1500 python bench.py --workload cfg4 --no-cpu-baseline --no-cold --steps 1 --warmup 1 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "cfg4=$?" >> $O/status.txt
timeout 1500 env HH_3D_MINB=3 python bench.py --workload cfg4 --no-cpu-baseline --no-cold --steps 1 --warmup 1 > $O/bench_cfg4_m3.json 2> $O/bench_cfg4_m3.err; echo "cfg4m3=$?" >> $O/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_march3d" -s 2 -c 1 -o $O/full_march_cfg4 python scripts/probe_3d.py cfg4 > $O/ncu.log 2>&1; echo "ncu=$?" >> $O/status.txt
