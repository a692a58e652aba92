timeout 900 python -m pytest tests/test_gpu_ttsvd.py tests/test_gpu_rank.py -x -q > gpurun_out/gputests_x.log 2>&1; echo "pytest rc $?"; tail -25 gpurun_out/gputests_x.log
