R=r64
timeout 900 python -m pytest tests/test_gpu_i8.py -q -x --timeout 600 -s 2>&1 | grep -E "rel-L2|passed|failed|Error" | tail -40
