# round-2 checkpoint 5 (top-k at copy bandwidth, eviction by latest use in the sharded scheduler, generalised persistent form):
# full GPU suite, smoke, the default bench line, reference arm, c3/c5 lines
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=8 > gpurun_out/r02ap_gputest.log 2>&1; echo "pytest rc=$?"; tail -14 gpurun_out/r02ap_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ap_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02ap_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r02ap_bench.log | head -c 2500; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02ap_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r02ap_ref.log | head -c 600; echo
for w in c1 c3 c5; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/r02ap_$w.log 2>&1; echo "[$w] rc=$?"; tail -1 gpurun_out/r02ap_$w.log | head -c 600; echo
done
