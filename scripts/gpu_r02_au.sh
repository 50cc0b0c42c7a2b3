#!/bin/bash
# 2D smoother tile shape: 32x16 (default) vs 32x32 vs 64x16 -- parity, per-size phases, sweep, cfg2
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02au
mkdir -p $O
for v in t32x32 t64x16; do
  HH_LIB=$PWD/paper_2104_01439_b200/libhh_$v.so timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_slabs.py > $O/pytest_$v.log 2>&1; echo "par_$v=$?" >> $O/status.txt
done
for v in default t32x32 t64x16; do
  L=""; [ $v != default ] && L="HH_LIB=$PWD/paper_2104_01439_b200/libhh_$v.so"
  env $L timeout 400 python scripts/probe_fd.py 68 268 534 > $O/probe_$v.txt 2>&1
  env $L timeout 400 python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/sweep_$v.json 2>/dev/null; echo "sweep_$v=$?" >> $O/status.txt
  env $L timeout 400 python bench.py --workload cfg2 --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/cfg2_$v.json 2>/dev/null; echo "cfg2_$v=$?" >> $O/status.txt
done
