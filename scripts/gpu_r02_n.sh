#!/bin/bash
# round 2: 3D pointwise streaming kernels + boundary faces on a side stream: parity + timing
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02n
mkdir -p $O
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_nd_forced.py tests/test_gpu_dist_coarse.py tests/test_gpu_flow.py tests/test_gpu_krylov_opts.py -k "not fullsize" > $O/pytest.log 2>&1; echo "par=$?" >> $O/status.txt
timeout 600 python scripts/probe_3d.py > $O/probe.json 2> $O/probe.err; echo "probe=$?" >> $O/status.txt
timeout 900 python bench.py --workload cfg3 --no-cpu-baseline --no-cold --steps 2 --warmup 2 > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo "cfg3=$?" >> $O/status.txt
timeout 900 env HH_3D_NOSIDE=1 python bench.py --workload cfg3 --no-cpu-baseline --no-cold --steps 2 --warmup 2 > $O/bench_cfg3_noside.json 2> $O/bench_cfg3_noside.err; echo "cfg3ns=$?" >> $O/status.txt
timeout 1500 python bench.py --workload cfg4 --no-cpu-baseline --no-cold --steps 1 --warmup 1 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "cfg4=$?" >> $O/status.txt
