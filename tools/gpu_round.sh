timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_bcd.py tests/test_gpu_dist.py tests/test_gpu_parity.py -q 2>&1 | tail -1
NTT_BCD_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bcd_c5b.csv python tools/bcd_c5_prof.py > /dev/null 2>&1; echo rc $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches5.csv python tools/prof_config5.py > /dev/null 2>&1; echo rc $?
timeout 600 python tools/bench_bcd.py config2 50 2>&1 | tail -1 | cut -c1-300
timeout 600 python tools/bench_bcd.py config5 20 2>&1 | tail -1 | cut -c1-300
