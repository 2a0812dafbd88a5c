B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fit --no-mlp --no-c3 --config c3"
$B > gpurun_out/plain_c3_pre.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pre3d -s 6 -c 2 -o gpurun_out/pre3d_c3 $B > gpurun_out/ncu_pre3d_c3.log 2>&1
tail -2 gpurun_out/ncu_pre3d_c3.log
