timeout 600 python -m pytest tests/test_gpu_bcd.py -q 2>&1 | tail -2
NTT_BCD_NO_1PASS=1 timeout 600 python -m pytest tests/test_gpu_bcd.py -q 2>&1 | tail -1
timeout 900 python tools/bench_bcd.py config2 20 sweep 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -1
