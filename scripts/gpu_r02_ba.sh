#!/bin/bash
# FD 40 x 40 tiles: parity + per-size probe + cfg3, with and without
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ba
mkdir -p $O
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_fd.py tests/test_gpu_goldens.py -k "not cfg4" > $O/pytest.log 2>&1; echo "par=$?" >> $O/status.txt
HH_FD_TILE=40 timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_fd.py > $O/pytest_force40.log 2>&1; echo "par40=$?" >> $O/status.txt
for u in 1 0; do
  HH_FD_TILE40=$u timeout 400 python scripts/probe_fd.py 134 400 468 534 > $O/probe_u$u.txt 2>&1
  HH_FD_TILE40=$u timeout 400 python bench.py --workload cfg3 --no-cpu-baseline --no-cold --steps 5 --warmup 3 > $O/cfg3_u$u.json 2>/dev/null
  HH_FD_TILE40=$u timeout 400 python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/sweep_u$u.json 2>/dev/null
done
