timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -1
timeout 300 python tools/bench_nmf.py config2 20 2>&1 | tail -1 > gpurun_out/c2_16.json
timeout 300 python tools/bench_nmf.py config5 5 2>&1 | tail -1 > gpurun_out/c5_16.json
