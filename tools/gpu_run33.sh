R=r33
for MIN in 1 64 512 4096; do
  PKGPU_M2L_I8_MIN=$MIN timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats > gpurun_out/${R}_min$MIN.log 2>&1
  echo "min=$MIN $(grep -E '^m2l ' gpurun_out/${R}_min$MIN.log | cut -c1-60) | $(grep -E '^m2l_i8 ' gpurun_out/${R}_min$MIN.log | cut -c1-50)"
done
