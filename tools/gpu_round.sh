set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_c -c 1 -o gpurun_out/fused_c_step2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-other > gpurun_out/ncu_fc.log 2>&1; echo "ncu rc $?"; tail -3 gpurun_out/ncu_fc.log
