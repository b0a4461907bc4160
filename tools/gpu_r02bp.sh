# round-2 final state: full GPU suite, smoke, default bench line, reference arm
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=8 > gpurun_out/r02bp_gputest.log 2>&1; echo "pytest rc=$?"; tail -14 gpurun_out/r02bp_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bp_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02bp_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r02bp_bench.log | head -c 600; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02bp_ref.log 2>&1; echo "ref rc=$?"
