timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -1
timeout 600 python bench.py --workload paper256 --steps 2 --warmup 1 --no-e2e --no-cpu --no-other > gpurun_out/bench_paper256.json 2> gpurun_out/bench_paper256.err; echo "rc $?"
python -c "
import json; d=json.load(open('gpurun_out/bench_paper256.json')); print(d['value'], d['ms_per_step'], d['config']['rel_error']); print({k: {kk: round(vv['ms_per_step'],2) for kk,vv in v.items()} for k,v in d['roofline']['per_tt_step'].items()})"
