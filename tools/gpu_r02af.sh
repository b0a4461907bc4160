# ncu --set full of a heavy (FP64-bound) persistent C4 pass: n=28, the 4th pass (175 FP64 per amplitude)
timeout 300 python tools/c4_once.py 28 10 > gpurun_out/r02af_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qcs_pass -s 3 -c 1 -o gpurun_out/r02af_c4heavy python tools/c4_once.py 28 10 > gpurun_out/r02af_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/r02af_ncu.log
