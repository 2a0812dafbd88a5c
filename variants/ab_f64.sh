bash variants/ab.sh base f64red f64mom > gpurun_out/ab_f64.txt 2>&1
WIPES_LIB=$PWD/variants/f64red.so timeout 300 python tools/diag_grad3d.py > gpurun_out/diag3d_f64red.log 2>&1
