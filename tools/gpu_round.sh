timeout 900 python -m pytest tests/test_gpu_bcd.py -q 2>&1 | tail -1
for i in 1 2; do timeout 600 python tools/bench_bcd.py config2 50 2>&1 | tail -1 | cut -c1-300; done
