#!/bin/bash
# FD root continuation with a loose intermediate tolerance: parity + setup timing (cfg3, sweep)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02at
mkdir -p $O
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_fd.py tests/test_gpu_goldens.py -k "not cfg4" > $O/pytest.log 2>&1; echo "par=$?" >> $O/status.txt
HH_PROFILE_SETUP=1 timeout 300 python bench.py --workload cfg3 --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/cfg3.json 2> $O/cfg3.err; echo "cfg3=$?" >> $O/status.txt
timeout 300 python bench.py --workload cfg3 --no-cpu-baseline --no-cold --steps 5 --warmup 3 > $O/cfg3b.json 2> $O/cfg3b.err
timeout 600 python bench.py --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/sweep.json 2>/dev/null; echo "sweep=$?" >> $O/status.txt
