#!/bin/bash
# persistent double-buffered constant-k pre-smoother (k_pre2d_pc) vs k_pre2d
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02az
mkdir -p $O
timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fd.py tests/test_gpu_slabs.py tests/test_gpu_goldens.py tests/test_gpu_krylov_opts.py -k "not cfg4" > $O/pytest.log 2>&1; echo "par=$?" >> $O/status.txt
timeout 400 python scripts/probe_fd.py 34 68 134 268 534 > $O/probe_p1.txt 2>&1
HH_FINE_PERSIST=0 timeout 400 python scripts/probe_fd.py 34 68 134 268 534 > $O/probe_p0.txt 2>&1
for i in 1 2; do
timeout 400 python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/sweep_p1_$i.json 2>/dev/null
HH_FINE_PERSIST=0 timeout 400 python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/sweep_p0_$i.json 2>/dev/null
done
