timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k small 2>&1 | tail -2
