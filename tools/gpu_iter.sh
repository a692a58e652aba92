python tools/prof_rk16.py 20 2>&1 | tail -4
python tools/pass_times.py 256 1048576 8 3 | head -3
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "mu" > gpurun_out/gputests_ab.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/gputests_ab.log
