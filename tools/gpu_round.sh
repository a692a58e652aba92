set -x
timeout 600 python -m pytest tests/test_gpu_bcd.py -q > gpurun_out/pytest_bcd.log 2>&1; echo "bcd rc $?"; grep -E "^E  |passed|failed" gpurun_out/pytest_bcd.log | head -30
