timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
timeout 300 python bench.py --workload config4 --steps 3 --warmup 3 --no-e2e --no-cpu --no-other 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('config4', d['ms_per_step'], d['config']['rel_error'])"
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-other 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('config3', d['ms_per_step'], d['config']['rel_error'], d['roofline']['frac'])"
