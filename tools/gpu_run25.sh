R=r25
timeout 300 python -m pytest tests/test_gpu_i8.py -q -x -k gather_gemm_exact 2>&1 | tail -15 > gpurun_out/${R}_i8gemm.log
cat gpurun_out/${R}_i8gemm.log
if grep -q "passed" gpurun_out/${R}_i8gemm.log && ! grep -q "failed" gpurun_out/${R}_i8gemm.log; then
  timeout 600 python -m pytest tests/test_gpu_i8.py -q 2>&1 | tail -25 > gpurun_out/${R}_i8all.log
  cat gpurun_out/${R}_i8all.log
  PKGPU_M2L=i8 timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats 2>&1 | grep -E "^m2l|timings|Error|error" > gpurun_out/${R}_stats.log
  cat gpurun_out/${R}_stats.log
  PKGPU_M2L=i8 PKGPU_M2L_I8_MIN=1 timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats 2>&1 | grep -E "^m2l|timings|Error|error" > gpurun_out/${R}_stats_all.log
  cat gpurun_out/${R}_stats_all.log
  PKGPU_M2L=i8 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}_ncu1.log 2>&1
  python tools/summarize_ncu.py launches gpurun_out/${R}_launches.csv --last-eval | head -12
fi
