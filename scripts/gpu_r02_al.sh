#!/bin/bash
# ND factorisation update with the 3M complex product: ND parity + cfg3 (ND forced) / cfg2 / cfg4 bench
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02al
mkdir -p $O
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_nd_forced.py tests/test_gpu_parity.py tests/test_gpu_goldens.py tests/test_gpu_dist_coarse.py tests/test_gpu_flow.py > $O/pytest.log 2>&1; echo "par=$?" >> $O/status.txt
timeout 600 python bench.py --workload cfg3 --coarse-solver nd --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/bench_cfg3_nd.json 2> $O/bench_cfg3_nd.err; echo "cfg3nd=$?" >> $O/status.txt
timeout 600 python bench.py --workload cfg2 --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "cfg2=$?" >> $O/status.txt
timeout 900 python bench.py --workload cfg4 --no-cpu-baseline --no-cold --steps 1 --warmup 1 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "cfg4=$?" >> $O/status.txt
