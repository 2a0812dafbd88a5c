timeout 600 python tools/sanitize_run.py 2d 3d next > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 2400 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize_run.py 2d 3d next > gpurun_out/memcheck.log 2>&1; echo "exit $?" >> gpurun_out/memcheck.log
