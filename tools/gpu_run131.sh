R=r131
for v in "4 64" "4 16" "8 64" "4 256" "2 64"; do set -- $v; PKGPU_GEMM_MINIT_SMALL=$1 PKGPU_GEMM_PART_MB=$2 python tools/run_cfg2.py --warm 3 --evals 10 --stats > gpurun_out/${R}_$1_$2.log 2>&1; echo "$v $(python tools/stage_ms.py gpurun_out/${R}_$1_$2.log 10 pinv_up pinv_dn m2m l2l)"; done
