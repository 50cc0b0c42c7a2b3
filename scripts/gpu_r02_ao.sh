#!/bin/bash
# column-strip stencil stages (FINE_COLS=1) vs the raster stages: parity + per-size phases + sweep
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ao
mkdir -p $O
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fd.py tests/test_gpu_slabs.py tests/test_gpu_goldens.py -k "not cfg4" > $O/pytest.log 2>&1; echo "par=$?" >> $O/status.txt
timeout 400 python scripts/probe_fd.py 68 268 534 > $O/probe_cols1.txt 2>&1
HH_LIB=$PWD/paper_2104_01439_b200/libhh_cols0.so timeout 400 python scripts/probe_fd.py 68 268 534 > $O/probe_cols0.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/sweep_cols1.json 2>/dev/null; echo "s1=$?" >> $O/status.txt
HH_LIB=$PWD/paper_2104_01439_b200/libhh_cols0.so timeout 600 python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/sweep_cols0.json 2>/dev/null; echo "s0=$?" >> $O/status.txt
