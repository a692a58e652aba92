timeout 600 python -m pytest tests/test_gpu_bcd.py -q 2>&1 | grep -E "^E  |passed|failed" | head -8
for i in 1 2; do timeout 900 python tools/bench_bcd.py config2 20 sweep 2>&1 | tail -2 | cut -c1-200; done
