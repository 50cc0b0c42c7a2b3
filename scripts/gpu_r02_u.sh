#!/bin/bash
# round 2: DMMA update on the small (32-row) tiles too: parity + A/B
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02u
mkdir -p $O
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_nd_forced.py tests/test_gpu_parity.py tests/test_gpu_sweep_share.py tests/test_gpu_flow.py > $O/pytest.log 2>&1; echo "par=$?" >> $O/status.txt
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_goldens.py > $O/pytest_goldens.log 2>&1; echo "gold=$?" >> $O/status.txt
for v in 2 1; do
  timeout 600 env HH_ND_MMA=$v python bench.py --no-cpu-baseline --no-cold --steps 2 --warmup 2 > $O/bench_sweep_mma$v.json 2> $O/bench_sweep_mma$v.err; echo "sweep_$v=$?" >> $O/status.txt
  timeout 600 env HH_ND_MMA=$v python bench.py --workload cfg2 --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/bench_cfg2_mma$v.json 2> $O/bench_cfg2_mma$v.err; echo "cfg2_$v=$?" >> $O/status.txt
  timeout 900 env HH_ND_MMA=$v python bench.py --workload cfg3 --no-cpu-baseline --no-cold --steps 2 --warmup 2 > $O/bench_cfg3_mma$v.json 2> $O/bench_cfg3_mma$v.err; echo "cfg3_$v=$?" >> $O/status.txt
done
