timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -k "decompose" 2>&1 | tail -8
