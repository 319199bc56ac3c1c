timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -rA --timeout 600 2>&1 | grep -E "rel-L2|passed|failed" 
for u in 4 8 16 32; do
  PKGPU_GEMM_UNITS=$u timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats 2>&1 | grep -E "^m2l" | sed "s/^/units=$u /"
done
