#!/bin/bash
# round 2, session 5: verify HEAD (full -m gpu suite, smoke, default bench, cfg2/cfg3 lines)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/s5a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=15 > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench exit $?" >> $O/bench_default.err
timeout 600 python bench.py --workload cfg2 --no-cpu-baseline --no-cold > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 600 python bench.py --workload cfg3 --no-cpu-baseline --no-cold > $O/bench_cfg3.json 2> $O/bench_cfg3.err
