R=r104
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -1
for E in 0 1; do
  if [ $E = 1 ]; then export PKGPU_GEMM_NOSMALL=1; fi
  timeout 300 python tools/run_cfg2.py --evals 6 --warm 2 --stats > gpurun_out/${R}_$E.log 2>&1
  python tools/stage_ms.py gpurun_out/${R}_$E.log 6 m2m l2l pinv_up pinv_dn
done
