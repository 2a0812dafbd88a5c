#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "c1_2d or mini or c2_kodak or c3 or more_than or c4 or c5" > gpurun_out/gpu_tests_sort4.log 2>&1
tail -2 gpurun_out/gpu_tests_sort4.log
for v in i12m3 i16m2; do
  WIPES_LIB=$PWD/variants/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "c1_2d or mini or c2_kodak or c3_full" > gpurun_out/gpu_tests_sort4_$v.log 2>&1
  echo "$v: $(tail -1 gpurun_out/gpu_tests_sort4_$v.log)"
done
bash variants/ab_sort.sh base i12m3 i16m2 i16m3 base > gpurun_out/ab_sort5.txt 2>&1
cat gpurun_out/ab_sort5.txt
