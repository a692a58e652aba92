timeout 600 python -m pytest tests -x -q -m gpu -k "nmf_mu or decompose or tc" 2>&1 | tail -2
timeout 300 python tools/prof_decompose.py config4 2 2>&1 | sed -n '1p;7,10p'
timeout 300 python tools/prof_decompose.py config1 2 2>&1 | head -1
