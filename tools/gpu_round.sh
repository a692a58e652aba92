timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_dist.py -q 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/c5_launches2.csv python tools/prof_config5.py > /dev/null 2>&1; echo rc $?
timeout 600 python tools/bench_nmf.py config5 10 2>&1 | tail -1 | cut -c1-300
