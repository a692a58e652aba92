timeout 600 python -m pytest tests/test_gpu_bcd.py tests/test_gpu_ttsvd.py -q -k "host" 2>&1 | grep -E "^E  |passed|failed" | head
