python tools/persist_trace.py > gpurun_out/ptrace_d.log 2>&1; cat gpurun_out/ptrace_d.log
python tools/tail_bench.py > gpurun_out/tail_d.log 2>&1; cat gpurun_out/tail_d.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_d.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/gputests_d.log
python bench.py --no-other --no-cpu > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err; echo "bench rc $?"
python -c "
import json;d=json.load(open('gpurun_out/bench_d.json'));r=d['roofline']
print(d['ms_per_step'], r['profiled_ms_per_step'], r['frac_of'], r['read_stream_ceiling_GBps'])
for k,v in r['per_tt_step'].items(): print(k, {a:(round(b['ms_per_step'],3), b['launches_per_step']) for a,b in v.items()})
"
