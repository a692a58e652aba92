timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_dist.py -x -q 2>&1 | tail -1
timeout 300 python tools/bench_nmf.py config2 20 2>&1 | tail -1 | cut -c1-200
timeout 300 python tools/bench_nmf.py config5 5 2>&1 | tail -1 | cut -c1-200
