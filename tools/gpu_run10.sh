mkdir -p gpurun_out/r10_ops
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r10_bench.json 2> gpurun_out/r10_bench.err
for e in "madelung1d --p-list 6,8" "laplace-dp-pair --p-list 8" "stokes-tp-dipole --p-list 8,10" "stokes-tp-force --p-list 8"; do
  timeout 600 ./oracle/_ref/pkifmm_dropin $e --operator-dir gpurun_out/r10_ops >> gpurun_out/r10_dropin.jsonl 2>> gpurun_out/r10_dropin.err; echo "rc=$? $e" >> gpurun_out/r10_dropin.jsonl
done
rm -rf gpurun_out/r10_ops
python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/r10_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r10_launches.csv python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/r10_ncu1.log 2>&1
cat gpurun_out/r10_bench.json; cat gpurun_out/r10_dropin.jsonl
