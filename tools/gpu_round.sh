timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_bcd.py tests/test_gpu_dist.py -q 2>&1 | tail -1
timeout 600 python tools/bench_nmf.py config5 10 2>&1 | tail -1 | cut -c1-600
timeout 600 python tools/bench_nmf.py config2 50 2>&1 | tail -1 | cut -c1-600
