R=r31
for D in 0 1 2 3 4 8 15; do
  PKGPU_I8_DEBUG=$D timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats > gpurun_out/${R}_dbg$D.log 2>&1
  echo "debug=$D $(grep -E '^m2l_i8' gpurun_out/${R}_dbg$D.log)"
done
