timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for c in config1 config3 config4; do timeout 300 python tools/prof_decompose.py $c 2 2>&1 | head -1; done
