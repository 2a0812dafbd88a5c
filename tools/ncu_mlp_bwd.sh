python paper_2508_12615_b200/build.py >/dev/null
timeout 120 python tools/bench_mlp.py 2>&1 | tail -c 300
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_mlp_bwd_layer -s 2 -c 1 -o gpurun_out/mlp_bwd_layer python tools/bench_mlp.py > gpurun_out/ncu_bwd.log 2>&1; echo ncu rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mlp2.csv python tools/bench_mlp.py > /dev/null 2>&1; echo rc=$?
