#!/bin/bash
# round 2: 2D smoothers staged with cp.async: A/B against register staging (-DFINE_ASYNC=0) + 2D parity
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02p
mkdir -p $O
C=paper_2104_01439_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -cudart shared \
  --expt-relaxed-constexpr -ldl -DFINE_ASYNC=0 -o /tmp/libhh_sync.so $C/hh_api.cu $C/fine2d.cu $C/fine3d.cu $C/coarse_nd.cu \
  $C/krylov.cu $C/comm.cu $C/lfa.cu $C/peak.cu > $O/build_sync.log 2>&1; echo "build=$?" >> $O/status.txt
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_flow.py tests/test_gpu_krylov_opts.py tests/test_gpu_sweep_share.py tests/test_gpu_search.py tests/test_gpu_slabs.py > $O/pytest_2d.log 2>&1; echo "par=$?" >> $O/status.txt
for impl in async sync; do
  if [ $impl = sync ]; then export HH_LIB=/tmp/libhh_sync.so; else unset HH_LIB; fi
  timeout 600 python bench.py --workload cfg2 --no-cpu-baseline --no-cold --steps 3 --warmup 3 > $O/bench_cfg2_$impl.json 2> $O/bench_cfg2_$impl.err; echo "cfg2_$impl=$?" >> $O/status.txt
  timeout 600 python bench.py --no-cpu-baseline --no-cold --steps 2 --warmup 2 > $O/bench_sweep_$impl.json 2> $O/bench_sweep_$impl.err; echo "sweep_$impl=$?" >> $O/status.txt
done
