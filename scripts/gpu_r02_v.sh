#!/bin/bash
# round 2 (session 4): full -m gpu suite with the HH_ND_MMA=2 default, smoke, bench lines, MMA A/B
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02v
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 2400 python -m pytest -q -p no:cacheprovider -m gpu tests --durations=30 > $O/pytest_gpu.log 2>&1; echo "gpu=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/status.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench=$?" >> $O/status.txt
for v in 2 1; do
  timeout 600 env HH_ND_MMA=$v python bench.py --workload cfg2 --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/bench_cfg2_mma$v.json 2> $O/bench_cfg2_mma$v.err; echo "cfg2_$v=$?" >> $O/status.txt
  timeout 900 env HH_ND_MMA=$v python bench.py --workload cfg3 --no-cpu-baseline --no-cold --steps 2 --warmup 2 > $O/bench_cfg3_mma$v.json 2> $O/bench_cfg3_mma$v.err; echo "cfg3_$v=$?" >> $O/status.txt
done
timeout 600 env HH_ND_MMA=1 python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/bench_sweep_mma1.json 2> $O/bench_sweep_mma1.err; echo "sweep_1=$?" >> $O/status.txt
