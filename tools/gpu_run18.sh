timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 600 2>&1 | grep -E "Error|error|assert|E  " | head -20
