timeout 600 python -m pytest tests/test_gpu_bcd.py -q 2>&1 | grep -E "^E  |passed|failed" | head -8
NTT_BCD_NO_CTA=1 timeout 600 python -m pytest tests/test_gpu_bcd.py -q 2>&1 | tail -1
timeout 600 python tools/bcd_steps.py 2>&1 | grep "bcd"
timeout 900 python tools/bench_bcd.py config2 20 sweep 2>&1 | tail -2 | cut -c1-200
