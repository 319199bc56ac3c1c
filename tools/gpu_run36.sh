R=r36
for C in 0 6 12 24; do
  PKGPU_I8_CHUNKS=$C timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats > gpurun_out/${R}_c$C.log 2>&1
  echo "chunks=$C $(grep -E '^m2l_i8 ' gpurun_out/${R}_c$C.log | cut -c1-50)"
done
PKGPU_I8_PAIR=3 PKGPU_I8_CHUNKS=12 timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats > gpurun_out/${R}_dual12.log 2>&1
echo "dual chunks=12 $(grep -E '^m2l_i8 ' gpurun_out/${R}_dual12.log | cut -c1-50)"
