timeout 600 python -m pytest tests/test_gpu_ttsvd.py -q -k "large_ranks" 2>&1 | grep -E "^E  |passed|failed" | head -8
