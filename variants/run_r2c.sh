bash variants/ab.sh base head > gpurun_out/ab_red.txt 2>&1
bash variants/run_sort.sh base s16 s12 lb8 > gpurun_out/ab_sort.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -s -p no:cacheprovider -k "c1_2d or tile_size or mini or partial or deterministic or forward_run or counters or c2_kodak" > gpurun_out/gpu_tests_red.log 2>&1
