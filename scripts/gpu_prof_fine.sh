# ncu --set full of the 2D fused fine kernels on cfg2 (heterogeneous) and a constant-k grid
mkdir -p gpurun_out/prof
for k in k_pre2d k_post2d; do
ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 1 -o gpurun_out/prof/fine_$k python scripts/ncu_target.py cfg2 > gpurun_out/prof/ncu_$k.log 2>&1
done
