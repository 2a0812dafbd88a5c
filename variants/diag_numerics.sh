set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/peaks_clocks.csv &
SMI=$!
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks tools/peaks.cu && /tmp/peaks gpurun_out/peaks.json > gpurun_out/peaks.txt 2>&1
kill $SMI
for v in WIPES_EXP_F64MOM WIPES_EXP_TRIG WIPES_EXP_F64MOM_WIPES_EXP_TRIG; do
  WIPES_LIB=$PWD/paper_2508_12615_b200/libwipes_$v.so timeout 300 python tools/diag_grad3d.py quick > gpurun_out/diag3d_$v.log 2>&1
done
