set -x
timeout 600 python -m pytest tests/test_gpu_ttsvd.py tests/test_gpu_rank.py -q 2>&1 | tail -2
timeout 600 python tools/bench_ttsvd.py config3 3 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ttsvd_launches2.csv python tools/bench_ttsvd.py config3 1 > gpurun_out/ncu_ttsvd.log 2>&1; echo "ncu rc $?"
