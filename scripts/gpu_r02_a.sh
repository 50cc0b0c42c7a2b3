#!/bin/bash
# round 2, first GPU pass: all -m gpu tests except the golden ones, then the default bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --ignore=tests/test_gpu_goldens.py -p no:cacheprovider \
  > gpurun_out/r02a/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02a/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 --records gpurun_out/r02a/sweep_records.jsonl \
  > gpurun_out/r02a/bench.json 2> gpurun_out/r02a/bench.err
echo "bench exit $?" >> gpurun_out/r02a/bench.err
