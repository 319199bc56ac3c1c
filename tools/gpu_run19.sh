timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -rA --timeout 600 2>&1 | grep -E "rel-L2|passed|failed"
