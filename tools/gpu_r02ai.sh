# ncu --set full of a C5-family pass at n=28 (relabelled pass, direct stores), checkpoint 4
timeout 300 python tools/c5_once.py 28 20 > gpurun_out/r02ai_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qcs_pass -s 8 -c 1 -o gpurun_out/r02ai_c5pass python tools/c5_once.py 28 20 > gpurun_out/r02ai_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/r02ai_ncu.log
