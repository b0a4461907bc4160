# persistent kernels: which shape fails under QCS_PERSIST=2 (C3 W3 rounds), and an ncu capture of the persistent C4 pass
for cfg in "c3 24" "c4 24" "c3 30"; do
  for e in "QCS_PERSIST=0" "QCS_PERSIST=2" "QCS_PERSIST=2 QCS_JIT_W4=0"; do
    env $e CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/persist_check.py $cfg 2>&1 | tail -2
  done
done
timeout 300 python tools/c4_once.py 28 10 > gpurun_out/r02ab_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qcs_pass -s 6 -c 1 -o gpurun_out/r02ab_c4pass python tools/c4_once.py 28 10 > gpurun_out/r02ab_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/r02ab_ncu.log
