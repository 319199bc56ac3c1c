R=r127
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -1
for m in 16 28 56; do PKGPU_GEMM_MINIT=$m python tools/run_cfg2.py --warm 3 --evals 10 --stats > gpurun_out/${R}_$m.log 2>&1; python tools/stage_ms.py gpurun_out/${R}_$m.log 10 m2l pinv_up pinv_dn m2m l2l tree lists leaf; done
