#!/bin/bash
# constant-k D^-1 division hoisted above the region loads in the 2D smoothers
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02bb
mkdir -p $O
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_slabs.py > $O/pytest.log 2>&1; echo "par=$?" >> $O/status.txt
timeout 400 python scripts/probe_fd.py 68 268 534 > $O/probe.txt 2>&1
for i in 1 2; do timeout 400 python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/sweep_$i.json 2>/dev/null; done
