#!/bin/bash
# one GPU round: full GPU suite, smoke, the default bench line, its ncu launch list, one
# `ncu --set full` capture each of the step-1 and step-2 kernels and the error-pass kernel (each ncu run only after the plain
# run exits 0), and the bench with the full config-4 oracle timing
cd "$(dirname "$0")/.." || exit 1
tag=${1:-r2}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_$tag.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/gputests_$tag.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; rc=$?; echo "bench rc $rc"
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-other \
    > gpurun_out/ncu_launch_$tag.log 2>&1; echo "ncu launches rc $?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_m -c 1 -f \
    -o gpurun_out/fused_m_$tag python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-other \
    > gpurun_out/ncu_full_m_$tag.log 2>&1; echo "ncu full m rc $?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_c -c 1 -f \
    -o gpurun_out/fused_c_$tag python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-other \
    > gpurun_out/ncu_full_c_$tag.log 2>&1; echo "ncu full c rc $?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tt_err -c 1 -f \
    -o gpurun_out/tt_err_$tag python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-other \
    > gpurun_out/ncu_full_tterr_$tag.log 2>&1; echo "ncu full tt_err rc $?"
fi
if [ -n "$2" ]; then
  timeout 1200 python bench.py --oracle-full --steps 2 --warmup 3 > gpurun_out/bench_oraclefull_$tag.json 2> gpurun_out/bench_oraclefull_$tag.err; echo "oracle-full bench rc $?"
fi
