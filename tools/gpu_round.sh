timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
NTT_W_BN=64 timeout 300 python tools/persist_trace.py 2>&1 | head -1
timeout 600 python bench.py --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']); print({k:round(list(v.values())[0]['ms_per_step'],2) for k,v in d['roofline']['per_tt_step'].items()})"
