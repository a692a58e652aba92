timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_dist.py tests/test_gpu_parity.py tests/test_gpu_rank.py -q 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches4.csv python tools/prof_config5.py > /dev/null 2>&1; echo rc $?
timeout 600 python tools/bench_bcd.py config5 20 2>&1 | tail -1 | cut -c1-400
timeout 600 python tools/bench_bcd.py config2 50 2>&1 | tail -1 | cut -c1-400
