#!/bin/bash
# one GPU round: full GPU suite, the default bench line, its ncu launch list and one
# `ncu --set full` capture of the dominant kernel (each ncu run only after the plain run exits 0)
cd "$(dirname "$0")/.." || exit 1
tag=${1:-r2}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_$tag.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/gputests_$tag.log
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; rc=$?; echo "bench rc $rc"
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-other \
    > gpurun_out/ncu_launch_$tag.log 2>&1; echo "ncu launches rc $?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 1 -f \
    -o gpurun_out/fused_$tag python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-other \
    > gpurun_out/ncu_full_$tag.log 2>&1; echo "ncu full rc $?"
fi
