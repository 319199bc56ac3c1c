R=r35
for P in 3 0; do
  PKGPU_I8_PAIR=$P timeout 120 python -m pytest tests/test_gpu_i8.py -q -x 2>&1 | tail -3 > gpurun_out/${R}_t$P.log; echo "pair=$P tests: $(tail -1 gpurun_out/${R}_t$P.log)"
  PKGPU_I8_PAIR=$P timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats > gpurun_out/${R}_stats_pair$P.log 2>&1
  echo "pair=$P $(grep -E '^m2l_i8' gpurun_out/${R}_stats_pair$P.log)"
done
