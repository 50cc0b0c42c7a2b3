#!/bin/bash
# round 2 (session 4): fast-diagonalisation coarse solve -- parity + first bench lines
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02w
mkdir -p $O
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_fd.py --durations=10 > $O/pytest_fd.log 2>&1; echo "fd=$?" >> $O/status.txt
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py > $O/pytest_parity.log 2>&1; echo "par=$?" >> $O/status.txt
timeout 600 python bench.py --no-cpu-baseline --no-cold --steps 2 --warmup 2 > $O/bench_sweep.json 2> $O/bench_sweep.err; echo "sweep=$?" >> $O/status.txt
timeout 600 python bench.py --workload cfg3 --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo "cfg3=$?" >> $O/status.txt
timeout 600 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_goldens.py tests/test_gpu_flow.py tests/test_gpu_nd_forced.py > $O/pytest_gold.log 2>&1; echo "gold=$?" >> $O/status.txt
