export WIPES_LIB=$PWD/variants/checks.so
timeout 900 python tools/sanitize_run.py 2d 3d next > gpurun_out/checks_sanitize.log 2>&1; echo "exit $?" >> gpurun_out/checks_sanitize.log
timeout 2400 python -m pytest tests/test_gpu_parity.py -q -s -p no:cacheprovider > gpurun_out/checks_parity.log 2>&1; echo "exit $?" >> gpurun_out/checks_parity.log
unset WIPES_LIB
timeout 900 python -m pytest tests/test_gpu_mlp.py -q -s -p no:cacheprovider -k "parity or image" > gpurun_out/gpu_tests_mlp.log 2>&1
bash variants/run_sort.sh base s4 s6 > gpurun_out/ab_sort2.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-c3 --no-fit > gpurun_out/bench_mlp.json 2> gpurun_out/bench_mlp.err
