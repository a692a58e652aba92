set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 2 -o gpurun_out/bench_full python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_full_bench.log 2>&1; echo "ncu full rc $?"
