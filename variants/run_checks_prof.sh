export WIPES_LIB=$PWD/variants/checks.so
timeout 900 python tools/sanitize_run.py 2d 3d next > gpurun_out/checks_sanitize.log 2>&1; echo "exit $?" >> gpurun_out/checks_sanitize.log
timeout 2400 python -m pytest tests/test_gpu_parity.py -q -s -p no:cacheprovider -x > gpurun_out/checks_parity.log 2>&1; echo "exit $?" >> gpurun_out/checks_parity.log
unset WIPES_LIB
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fit --no-mlp --no-c3"
$B > gpurun_out/plain_c2.log 2>&1 && $B --config c3 > gpurun_out/plain_c3.log 2>&1 && $B --config c5 > gpurun_out/plain_c5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $B > /dev/null 2>&1 ; \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $B --config c3 > /dev/null 2>&1 ; \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv $B --config c5 > /dev/null 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:k_render -s 12 -c 2 -o gpurun_out/rend_c2_r02 $B > /dev/null 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:"k_render|k_sort_pass" -s 20 -c 3 -o gpurun_out/rend_c3_r02 $B --config c3 > /dev/null 2>&1
