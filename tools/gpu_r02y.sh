# round-2: every workload's bench line after the round-2 planner (c1, c2, c3, c5-shaped n=32, rh-signs), C5 launch list + one full capture
for w in c1 c3 c5 rh-signs; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/r02y_$w.log 2>&1; echo "[$w] rc=$?"; tail -1 gpurun_out/r02y_$w.log | head -c 1200; echo
done
timeout 900 python bench.py --workload c2 --steps 3 --warmup 3 > gpurun_out/r02y_c2.log 2>&1; echo "[c2] rc=$?"; tail -1 gpurun_out/r02y_c2.log | head -c 1200; echo
timeout 300 python tools/c5_once.py 32 20 > gpurun_out/r02y_c5once.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02y_c5_launches.csv python tools/c5_once.py 32 20 > gpurun_out/r02y_ncu1.log 2>&1; echo "ncu launches rc=$?"
timeout 300 python tools/c5_once.py 28 20 > gpurun_out/r02y_c5once28.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:qcs_pass -s 3 -c 1 -o gpurun_out/r02y_c5_full python tools/c5_once.py 28 20 > gpurun_out/r02y_ncu2.log 2>&1; echo "ncu full rc=$?"
