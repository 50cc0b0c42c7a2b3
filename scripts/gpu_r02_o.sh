#!/bin/bash
# round 2: full-size goldens (cfg1 all samples, cfg2, cfg3) + distributed coarse at full size
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02o
mkdir -p $O
timeout 2400 python -m pytest -q -p no:cacheprovider tests/test_gpu_goldens.py -k "cfg1 or cfg2 or cfg3" > $O/pytest_goldens.log 2>&1; echo "gold=$?" >> $O/status.txt
timeout 2400 env HH_DEBUG=1 python -m pytest -q -p no:cacheprovider tests/test_gpu_dist_coarse.py -k fullsize > $O/pytest_distfull.log 2>&1; echo "distfull=$?" >> $O/status.txt
