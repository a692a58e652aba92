set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; grep -E "^E  |passed|failed" gpurun_out/pytest_gpu.log | head -30
timeout 600 python tools/bench_nmf.py config2 50 2>&1 | tail -2
timeout 600 python tools/bench_nmf.py config5 10 2>&1 | tail -2
timeout 600 python tools/bench_bcd.py config2 50 2>&1 | tail -3
