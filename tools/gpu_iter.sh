timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/gputests_n.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/gputests_n.log
python tools/dist1_overhead.py > gpurun_out/dist1_n.log 2>&1; cat gpurun_out/dist1_n.log
