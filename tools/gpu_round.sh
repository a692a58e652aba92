set -x
timeout 600 python -m pytest tests/test_gpu_bcd.py -q > gpurun_out/pytest_bcd.log 2>&1; echo "bcd rc $?"; grep -E "^E  |passed|failed" gpurun_out/pytest_bcd.log | head -30
NTT_NO_TC=1 timeout 600 python -m pytest tests/test_gpu_bcd.py -q 2>&1 | tail -3
NTT_BCD_GRAPH=0 timeout 600 python -m pytest tests/test_gpu_bcd.py -q 2>&1 | tail -3
timeout 600 python tools/bench_bcd.py config2 50 2>&1 | tail -3
timeout 600 python tools/bench_bcd.py config5 20 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bcd_launches.csv python tools/bench_bcd.py config2 3 > gpurun_out/ncu_bcd.log 2>&1; echo "ncu rc $?"
