#!/bin/bash
# compute-sanitizer memcheck and racecheck on the 2D paths (C1-sized inputs)
python paper_2508_12615_b200/build.py > /dev/null || exit 1
which compute-sanitizer; compute-sanitizer --version | tail -1
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize_run.py 2d > gpurun_out/memcheck_2d.log 2>&1; echo "memcheck exit $?" | tee -a gpurun_out/memcheck_2d.log
tail -5 gpurun_out/memcheck_2d.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/sanitize_run.py 2d > gpurun_out/racecheck_2d.log 2>&1; echo "racecheck exit $?" | tee -a gpurun_out/racecheck_2d.log
tail -5 gpurun_out/racecheck_2d.log
