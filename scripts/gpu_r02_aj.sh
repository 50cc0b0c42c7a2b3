#!/bin/bash
# FD 3M complex product: parity + per-size probe + sweep/cfg3 bench
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02aj
mkdir -p $O
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_fd.py tests/test_gpu_parity.py tests/test_gpu_goldens.py > $O/pytest.log 2>&1; echo "par=$?" >> $O/status.txt
timeout 400 python scripts/probe_fd.py > $O/probe_fd.txt 2>&1; echo "probe=$?" >> $O/status.txt
timeout 600 python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/bench_sweep.json 2> $O/bench_sweep.err; echo "sweep=$?" >> $O/status.txt
timeout 600 python bench.py --workload cfg3 --no-cpu-baseline --no-cold --steps 5 --warmup 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo "cfg3=$?" >> $O/status.txt
