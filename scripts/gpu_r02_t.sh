#!/bin/bash
# round 2: pivot blocks of 64 with the DMMA update: parity (forced on small fronts) + A/B
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02t
mkdir -p $O
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_nd_forced.py tests/test_gpu_parity.py > $O/pytest.log 2>&1; echo "par=$?" >> $O/status.txt
for v in 1073741824 4096 2048; do
  timeout 900 env HH_ND_NB64_F=$v HH_PROFILE_SETUP=2 python scripts/probe_cfg3.py cfg3 > $O/factor_cfg3_nb64_$v.txt 2>&1; echo "prof_$v=$?" >> $O/status.txt
done
