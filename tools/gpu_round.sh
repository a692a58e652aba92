timeout 600 python -m pytest tests/test_gpu_bcd.py tests/test_gpu_parity.py -q 2>&1 | tail -1
timeout 900 python tools/bench_bcd.py config2 20 sweep 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-other 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']['per_tt_step']; print('config3', d['ms_per_step'], d['roofline']['frac'], [round(r[k]['xstream']['ms_per_step'],2) for k in r if 'xstream' in r[k]])"; done
