timeout 900 python -m pytest tests/test_gpu_bcd.py -q 2>&1 | grep -E "^E  |passed|failed" | head -6
timeout 600 python tools/bcd_steps4.py 2>&1 | grep bcd
NTT_BCD_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bcd_small2.csv python tools/bcd_small_prof.py > /dev/null 2>&1; echo rc $?
