R=r38
for E in transpose direct; do
  PKGPU_I8_EPI=$E timeout 120 python -m pytest tests/test_gpu_i8.py -q -x 2>&1 | tail -2 > gpurun_out/${R}_t$E.log; echo "epi=$E tests: $(tail -1 gpurun_out/${R}_t$E.log)"
  for C in 0 6; do
    PKGPU_I8_EPI=$E PKGPU_I8_CHUNKS=$C timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats > gpurun_out/${R}_${E}_c$C.log 2>&1
    echo "epi=$E chunks=$C $(grep -E '^m2l_i8 ' gpurun_out/${R}_${E}_c$C.log | cut -c1-50)"
  done
done
