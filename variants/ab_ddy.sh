bash variants/ab.sh base ddy ddyred > gpurun_out/ab_ddy.txt 2>&1
for v in ddy ddyred; do WIPES_LIB=$PWD/variants/$v.so timeout 300 python tools/diag_grad3d.py > gpurun_out/diag3d_$v.log 2>&1; done
