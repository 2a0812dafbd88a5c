bash variants/ab.sh base head f32all xprod > gpurun_out/ab_accum.txt 2>&1
timeout 300 python tools/diag_grad3d.py > gpurun_out/diag3d_new.log 2>&1
WIPES_LIB=$PWD/variants/xprod.so timeout 300 python tools/diag_grad3d.py quick > gpurun_out/diag3d_xprod.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
free -g > gpurun_out/free.txt; nproc >> gpurun_out/free.txt
