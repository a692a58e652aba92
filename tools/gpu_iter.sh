python tools/prof_rk16.py 20 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/gputests_q.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/gputests_q.log
python bench.py --no-other --no-cpu > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc $?"
python -c "
import json;d=json.load(open('gpurun_out/bench_q.json'));r=d['roofline']
print(d['ms_per_step'], r['profiled_ms_per_step'], r['frac_of'], d['clocks'])
for k,v in r['per_tt_step'].items(): print(k, {a:(round(b['ms_per_step'],3), b['launches_per_step']) for a,b in v.items()})
"
