timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/gputests_af.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/gputests_af.log
