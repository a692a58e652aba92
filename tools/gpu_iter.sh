timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_o.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/gputests_o.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_o.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/smoke_o.log
python bench.py --no-other --no-cpu --workload config4 > gpurun_out/bench_c4_o.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/bench_c4_o.json'));print('config4', d['ms_per_step'])"
