timeout 300 python tools/persist_trace.py 2>&1 | tail -8
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python tools/prof_decompose.py config3 2 2>&1 | head -7
timeout 300 python tools/prof_decompose.py config4 2 2>&1 | head -1
timeout 300 python tools/prof_decompose.py config1 2 2>&1 | head -1
