timeout 600 python -m pytest tests/test_gpu_bcd.py -q 2>&1 | grep -E "^E  |passed|failed" | head -8
NTT_BCD_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bcd_s1b.csv python tools/bcd_step1_prof.py > /dev/null 2>&1; echo rc $?
timeout 600 python tools/bcd_steps.py 2>&1 | grep "bcd"
timeout 900 python tools/bench_bcd.py config2 20 sweep 2>&1 | tail -2 | cut -c1-200
