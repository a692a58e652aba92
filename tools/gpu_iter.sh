timeout 900 python -m pytest tests/test_gpu_rank.py -x -q > gpurun_out/gputests_k.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/gputests_k.log
python tools/eps_sweep.py > gpurun_out/eps_sweep_r2.md 2> gpurun_out/eps_sweep_r2.err; echo "rc $?"; cat gpurun_out/eps_sweep_r2.md; tail -3 gpurun_out/eps_sweep_r2.err
