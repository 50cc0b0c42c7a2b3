#!/bin/bash
# round 2: DMMA (FP64 tensor path) factor update: parity + A/B
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02r
mkdir -p $O
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_nd_forced.py tests/test_gpu_dist_coarse.py tests/test_gpu_slabs.py -k "not fullsize" > $O/pytest.log 2>&1; echo "par=$?" >> $O/status.txt
timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_goldens.py -k "cfg2 or cfg3" > $O/pytest_goldens.log 2>&1; echo "gold=$?" >> $O/status.txt
timeout 600 env HH_PROFILE_SETUP=2 python scripts/probe_cfg3.py cfg3 > $O/factor_levels_cfg3_mma.txt 2>&1; echo "prof=$?" >> $O/status.txt
for v in 1 0; do
  timeout 900 env HH_ND_MMA=$v python bench.py --workload cfg3 --no-cpu-baseline --no-cold --steps 2 --warmup 2 > $O/bench_cfg3_mma$v.json 2> $O/bench_cfg3_mma$v.err; echo "cfg3_$v=$?" >> $O/status.txt
  timeout 600 env HH_ND_MMA=$v python bench.py --no-cpu-baseline --no-cold --steps 2 --warmup 2 > $O/bench_sweep_mma$v.json 2> $O/bench_sweep_mma$v.err; echo "sweep_$v=$?" >> $O/status.txt
done
timeout 1500 python bench.py --workload cfg4 --no-cpu-baseline --no-cold --steps 1 --warmup 1 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "cfg4=$?" >> $O/status.txt
