timeout 1200 python tools/eps256.py > gpurun_out/eps256.md 2> gpurun_out/eps256.err; echo "rc $?"; cat gpurun_out/eps256.md; tail -3 gpurun_out/eps256.err
