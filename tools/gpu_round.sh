timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -k "bcd_config5 or ttsvd_config3" 2>&1 | grep -E "^E  |passed|failed" | head -10
