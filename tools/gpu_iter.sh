python bench.py --workload config1 --no-other --no-cpu --no-e2e > gpurun_out/bench_c1_s.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/bench_c1_s.json'));r=d['roofline']
print('config1', d['ms_per_step'])
for k,v in r['per_tt_step'].items(): print(k, {a:(round(b['ms_per_step'],3), b['launches_per_step']) for a,b in v.items()})"
python tools/tail_bench.py 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/gputests_s.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/gputests_s.log
