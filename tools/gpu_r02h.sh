# compute-sanitizer memcheck over every kernel family (tools/sanitize_run.py), after a plain run
timeout 300 python tools/sanitize_run.py > gpurun_out/r02h_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_run.py > gpurun_out/r02h_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -6 gpurun_out/r02h_memcheck.log; tail -3 gpurun_out/r02h_plain.log
