timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
timeout 300 python tools/persist_trace.py 2>&1 | sed -n 2,3p
timeout 300 python tools/persist_trace.py 2>&1 | sed -n 2,3p
