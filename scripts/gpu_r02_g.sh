#!/bin/bash
# round 2: 3D kernel A/B (naive vs z-marching, 2 vs 3 CTAs/SM) + distributed coarse at scale
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02g
mkdir -p $O
timeout 600 python scripts/probe_3d.py > $O/probe_march3.json 2> $O/probe_march3.err; echo "m3=$?" >> $O/status.txt
timeout 600 env HH_3D_MINB=2 python scripts/probe_3d.py > $O/probe_march2.json 2> $O/probe_march2.err; echo "m2=$?" >> $O/status.txt
timeout 600 env HH_3D_NAIVE=1 python scripts/probe_3d.py > $O/probe_naive.json 2> $O/probe_naive.err; echo "naive=$?" >> $O/status.txt
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_dist_coarse.py tests/test_gpu_parity.py -k "dist or cfg3 or cfg4" > $O/pytest_dist.log 2>&1; echo "dist=$?" >> $O/status.txt
