#!/bin/bash
# session 6: ncu --set full captures of the fused 2D smoothers (sweep n = 534 batches, cfg2) and the 3D z-marching
# kernels (cfg3 constant k, cfg4 medium at 129^3 heterogeneous) at HEAD; 5 repeats of the default bench (spread)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02s6c; mkdir -p $O
for i in 1 2 3 4 5; do
  timeout 300 python bench.py --no-cpu-baseline --no-cold 2>>$O/err.log | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'value': d['value'], 'ms_per_step': d['ms_per_step'], 'e2e': d['e2e']['value'], 'krylov_frac': d['roofline']['frac'], 'clocks': d['clocks']}))" >> $O/bench_repeats.jsonl
done
for k in k_pre2d k_post2d; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 300 -c 1 -o $O/full_sweep534_$k \
    python scripts/probe_fd.py 534 > $O/ncu_sweep534_$k.log 2>&1; echo "sweep_$k=$?" >> $O/status.txt
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 1 -o $O/full_cfg2_$k \
    python scripts/ncu_target.py cfg2 > $O/ncu_cfg2_$k.log 2>&1; echo "cfg2_$k=$?" >> $O/status.txt
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_march3d -s 40 -c 8 -o $O/full_cfg3_k_march3d \
  python scripts/probe_cfg3.py cfg3 > $O/ncu_cfg3_march.log 2>&1; echo "cfg3_march=$?" >> $O/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_march3d -s 40 -c 8 -o $O/full_cfg4m_k_march3d \
  python scripts/probe_cfg3.py cfg4 128 > $O/ncu_cfg4m_march.log 2>&1; echo "cfg4m_march=$?" >> $O/status.txt
