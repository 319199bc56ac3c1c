python tools/run_cfg2.py --evals 2 --stats > gpurun_out/r3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_launches.csv python tools/run_cfg2.py --evals 1 > gpurun_out/r3_ncu1.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:gather_gemm_kernel -s 28 -c 1 -o gpurun_out/r3_m2l python tools/run_cfg2.py --evals 1 > gpurun_out/r3_ncu2.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:leaf_kernel -c 1 -o gpurun_out/r3_leaf python tools/run_cfg2.py --evals 1 > gpurun_out/r3_ncu3.log 2>&1; \
tail -3 gpurun_out/r3_ncu2.log
