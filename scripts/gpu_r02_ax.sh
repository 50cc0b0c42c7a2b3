#!/bin/bash
# evidence pass after the stream / sharding / FD-tolerance changes
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ax
mkdir -p $O
timeout 2400 python -m pytest -q -p no:cacheprovider -m gpu tests --durations=10 > $O/pytest_gpu.log 2>&1; echo "gpu=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/status.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench=$?" >> $O/status.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-cold > $O/bench_sweep_k5.json 2> $O/bench_sweep_k5.err; echo "bench5=$?" >> $O/status.txt
