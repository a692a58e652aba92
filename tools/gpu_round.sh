set -x
timeout 600 python -m pytest tests/test_gpu_ttsvd.py -q > gpurun_out/pytest_ttsvd.log 2>&1; echo "ttsvd rc $?"; grep -E "^E  |passed|failed|Error" gpurun_out/pytest_ttsvd.log | head -40
