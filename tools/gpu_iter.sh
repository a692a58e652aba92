timeout 900 python -m pytest tests/test_gpu_bcd.py -x -q > gpurun_out/gputests_z.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/gputests_z.log
