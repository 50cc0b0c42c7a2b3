#!/bin/bash
# Krylov update in reverse CTA order (L2 reuse of the multi-dot's last chunks): parity + probe + sweep
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ay
mkdir -p $O
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_krylov_opts.py tests/test_gpu_slabs.py > $O/pytest.log 2>&1; echo "par=$?" >> $O/status.txt
timeout 400 python scripts/probe_fd.py 134 268 534 > $O/probe_rev1.txt 2>&1
HH_LIB=$PWD/paper_2104_01439_b200/libhh_rev0.so timeout 400 python scripts/probe_fd.py 134 268 534 > $O/probe_rev0.txt 2>&1
for i in 1 2; do
timeout 400 python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/sweep_rev1_$i.json 2>/dev/null
HH_LIB=$PWD/paper_2104_01439_b200/libhh_rev0.so timeout 400 python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/sweep_rev0_$i.json 2>/dev/null
done
timeout 400 python bench.py --workload cfg2 --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/cfg2_rev1.json 2>/dev/null
HH_LIB=$PWD/paper_2104_01439_b200/libhh_rev0.so timeout 400 python bench.py --workload cfg2 --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/cfg2_rev0.json 2>/dev/null
