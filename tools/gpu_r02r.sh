# ncu --set full of one C4 fused pass (n=28, 10 layers), end of round 2 (TMA-preferring tiles)
timeout 300 python tools/c4_once.py 28 10 > gpurun_out/r02r_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qcs_pass -s 6 -c 1 -o gpurun_out/r02r_c4pass python tools/c4_once.py 28 10 > gpurun_out/r02r_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/r02r_ncu.log
