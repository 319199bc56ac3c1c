R=r41
run() { timeout 300 python tools/run_cfg2.py --evals 6 --warm 2 --stats > gpurun_out/${R}_$1.log 2>&1; echo "$1 $(grep -E '^m2l_i8 ' gpurun_out/${R}_$1.log | cut -c1-48)"; }
run base
PKGPU_I8_DEBUG=16 run oneop
PKGPU_I8_PREFETCH=4 run pf4
PKGPU_I8_PREFETCH=8 run pf8
PKGPU_I8_PREFETCH=16 run pf16
run base2
