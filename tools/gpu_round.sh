timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "256 or 200 or 100 or 64 or 41" 2>&1 | tail -1
for i in 1 2; do timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-other 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']['per_tt_step']; print('config3', d['ms_per_step'], d['roofline']['frac'], [round(r[k]['xstream']['ms_per_step'],2) for k in r if 'xstream' in r[k]])"; done
