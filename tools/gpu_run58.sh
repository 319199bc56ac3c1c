R=r58
# full capture of the cfg2 level-4 M2L launch (2nd m2l_i8 launch of the profiled eval), single and dual
timeout 900 ncu --set full --import-source on --clock-control none -k regex:m2l_i8_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/${R}_single python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}_single.log 2>&1
PKGPU_I8_PAIR=3 timeout 900 ncu --set full --import-source on --clock-control none -k regex:m2l_i8_dual --launch-skip 3 --launch-count 1 -o gpurun_out/${R}_dual python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}_dual.log 2>&1
ls -la gpurun_out/
