timeout 900 python -m pytest tests/test_gpu_partition.py -q -x --timeout 600 -k adaptive 2>&1 | grep -E "assert|Error|rel|E  " | head -20
