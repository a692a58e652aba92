timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
timeout 120 python tools/prof_decompose.py config4 2 2>&1 | sed -n 1,4p
timeout 120 python tools/prof_decompose.py config3 2 2>&1 | sed -n 1,3p
