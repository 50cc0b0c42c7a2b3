#!/bin/bash
# ND 3M update with the epilogue loads batched: forced-ND parity + cfg3 (ND) / cfg2 bench
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02am
mkdir -p $O
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_nd_forced.py > $O/pytest.log 2>&1; echo "par=$?" >> $O/status.txt
timeout 600 python bench.py --workload cfg3 --coarse-solver nd --no-cpu-baseline --no-cold --steps 3 --warmup 2 > $O/bench_cfg3_nd.json 2> $O/bench_cfg3_nd.err; echo "cfg3nd=$?" >> $O/status.txt
timeout 600 python bench.py --workload cfg2 --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "cfg2=$?" >> $O/status.txt
