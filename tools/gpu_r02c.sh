# round-2 GPU check: the new tests (sampling, shims, dumps, BASELINE sizes with the threaded oracle)
nproc
timeout 1500 python -m pytest -q tests/test_sample_gpu.py tests/test_shim_gpu.py tests/test_jit.py tests/test_baseline_sizes_gpu.py "tests/test_parity_gpu.py::test_encoder_bytes_vs_oracle_and_golden" "tests/test_parity_gpu.py::test_dumps_vs_live_reference" tests/test_circuit_io.py -m gpu -rs --durations=12 -s > gpurun_out/r02c_tests.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|shim|python_kept" gpurun_out/r02c_tests.log | tail -5; tail -22 gpurun_out/r02c_tests.log
