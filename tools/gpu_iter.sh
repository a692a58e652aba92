timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_bcd.py -x -q > gpurun_out/gputests_w.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/gputests_w.log
python bench.py --no-other --no-cpu > gpurun_out/bench_w.json 2> gpurun_out/bench_w.err; echo "bench rc $?"
python -c "
import json;d=json.load(open('gpurun_out/bench_w.json'));r=d['roofline']
print(d['ms_per_step'], r['profiled_ms_per_step'], r['frac_of'], d['clocks'])
for k,v in r['per_tt_step'].items(): print(k, {a:(round(b['ms_per_step'],3), b['launches_per_step']) for a,b in v.items()})
"
python bench.py --workload paper256 --no-other --no-cpu --no-e2e --steps 2 --warmup 3 > gpurun_out/bench_p256_w.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/bench_p256_w.json'));r=d['roofline']
print('paper256', d['ms_per_step'])
for k,v in r['per_tt_step'].items(): print(k, {a:(round(b['ms_per_step'],3), b['launches_per_step']) for a,b in v.items()})"
