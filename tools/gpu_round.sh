set -x
timeout 600 python -m pytest tests/test_gpu_bcd.py -x -q > gpurun_out/pytest_bcd.log 2>&1; echo "bcd rc $?"; tail -30 gpurun_out/pytest_bcd.log
