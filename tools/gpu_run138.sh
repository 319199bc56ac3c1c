timeout 1200 python -m pytest tests/test_gpu_i8.py -q -x -k "pair_dual" 2>&1 | tail -3
