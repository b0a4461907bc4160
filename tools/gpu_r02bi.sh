# round-2 final: full GPU suite, smoke, default bench line, reference arm (after the sharded-path and cold-start changes)
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=8 > gpurun_out/r02bi_gputest.log 2>&1; echo "pytest rc=$?"; tail -14 gpurun_out/r02bi_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bi_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02bi_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r02bi_bench.log | head -c 1500; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02bi_ref.log 2>&1; echo "ref rc=$?"
timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/r02bi_c5.log 2>&1; echo "[c5] rc=$?"; tail -1 gpurun_out/r02bi_c5.log | head -c 300; echo
