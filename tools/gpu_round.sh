set -x
timeout 600 python -m pytest tests/test_gpu_bcd.py -q > gpurun_out/pytest_bcd.log 2>&1; echo "bcd rc $?"; grep -E "^E  |passed|failed" gpurun_out/pytest_bcd.log | head -30
NTT_BCD_NO_FUSED=1 timeout 600 python -m pytest tests/test_gpu_bcd.py -q 2>&1 | tail -2
NTT_NO_TC=1 timeout 600 python -m pytest tests/test_gpu_bcd.py -q 2>&1 | tail -2
timeout 900 python tools/bench_bcd.py config2 20 sweep 2>&1 | tail -3
