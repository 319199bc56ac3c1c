R=r82
timeout 900 python -m pytest tests/test_gpu_periodize.py -q -x -s --timeout 800 2>&1 | grep -E "rel|diff|passed|failed|Error|error|assert" | head -40
