timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -1
for ux in 5 1; do NTT_X3D_UX=$ux timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-other 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']['per_tt_step']; print('ux<=$ux', d['ms_per_step'], d['config']['rel_error'], d['roofline']['frac'], [round(r[k]['xstream']['ms_per_step'],2) for k in r if 'xstream' in r[k]])"; done
