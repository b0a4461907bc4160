timeout 300 python tools/nccl_self_exchange.py 29655 2>&1 | tail -6
timeout 600 python -m pytest -q tests/test_partition_gpu.py -m gpu -x 2>&1 | tail -3
