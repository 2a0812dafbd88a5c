nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks tools/peaks.cu && /tmp/peaks gpurun_out/peaks2.json > gpurun_out/peaks2.txt 2>&1
timeout 600 python tools/diag_grad3d.py > gpurun_out/diag3d_e1.log 2>&1
timeout 600 python tools/diag_grad3d.py seeds > gpurun_out/diag3d_e1_seeds.log 2>&1
WIPES_LIB=$PWD/variants/fprod.so timeout 300 python tools/diag_grad3d.py seeds > gpurun_out/diag3d_fprod_seeds.log 2>&1
bash variants/ab.sh base > gpurun_out/ab_e1.txt 2>&1
