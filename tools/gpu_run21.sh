timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats 2>&1 | grep -E "^m2l|timings|pkgpu|Error"
