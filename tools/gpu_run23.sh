R=r23
timeout 300 python -m pytest tests/test_gpu_i8.py -q -x -k gather_gemm_exact 2>&1 | tail -15 > gpurun_out/${R}_i8gemm.log
cat gpurun_out/${R}_i8gemm.log
if grep -q "passed" gpurun_out/${R}_i8gemm.log && ! grep -q "failed" gpurun_out/${R}_i8gemm.log; then
  timeout 600 python -m pytest tests/test_gpu_i8.py -q 2>&1 | tail -25 > gpurun_out/${R}_i8all.log
  cat gpurun_out/${R}_i8all.log
  timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats 2>&1 | grep -E "^m2l|timings|Error|error" > gpurun_out/${R}_stats.log
  cat gpurun_out/${R}_stats.log
  timeout 1200 python tools/quant_study.py --specs "dmma;q:56;q:52;i8:17,56,56;i8all:17,56,56;i8all:16,52,52;i8all:15,48,48" > gpurun_out/${R}_quant.jsonl 2>&1
  cat gpurun_out/${R}_quant.jsonl | cut -c1-400
fi
