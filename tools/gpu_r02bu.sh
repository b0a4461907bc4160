# ncu --set full of the final plan's heaviest C4 pass (the first full-size pass after the deferred part: 234.5 FP64 per amplitude) at n=28,
# and of a quarter-support pass (one tile per CTA, compact launch)
timeout 300 python tools/c4_once.py 28 10 > gpurun_out/r02bu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qcs_pass -s 6 -c 1 -o gpurun_out/r02bu_c4cone python tools/c4_once.py 28 10 > gpurun_out/r02bu_ncu.log 2>&1; echo "ncu cone rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qcs_pass -s 2 -c 1 -o gpurun_out/r02bu_c4quarter python tools/c4_once.py 28 10 > gpurun_out/r02bu_ncu2.log 2>&1; echo "ncu quarter rc=$?"
