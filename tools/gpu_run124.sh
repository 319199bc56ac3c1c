R=r124
for m in 16 8 4 2; do PKGPU_GEMM_MINIT_SMALL=$m python tools/run_cfg2.py --warm 3 --evals 10 --stats > gpurun_out/${R}_$m.log 2>&1; python tools/stage_ms.py gpurun_out/${R}_$m.log 10 m2l pinv_up pinv_dn m2m l2l; done
