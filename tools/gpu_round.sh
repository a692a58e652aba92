set -x
timeout 600 python -m pytest tests/test_gpu_bcd.py -q > gpurun_out/pytest_bcd.log 2>&1; echo "bcd rc $?"; grep -E "^E  |passed|failed" gpurun_out/pytest_bcd.log | head -30
timeout 900 python tools/bench_bcd.py config2 20 sweep 2>&1 | tail -3
timeout 900 python tools/bench_bcd.py config5 20 2>&1 | tail -1
