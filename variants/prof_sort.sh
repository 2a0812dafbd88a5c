B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fit --no-mlp --no-c3 --config c3"
$B > gpurun_out/plain_c3_sort.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sort_pass -s 42 -c 7 -o gpurun_out/sort_c3 $B > gpurun_out/ncu_sort_c3.log 2>&1
tail -3 gpurun_out/ncu_sort_c3.log
