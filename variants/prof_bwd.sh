B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fit --no-mlp --no-c3"
$B > gpurun_out/plain_c2.log 2>&1 && $B --config c3 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_render_bwd -s 6 -c 1 -o gpurun_out/bwd_c2 $B > gpurun_out/ncu_c2.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:k_render_bwd -s 6 -c 1 -o gpurun_out/bwd_c3 $B --config c3 > gpurun_out/ncu_c3.log 2>&1
