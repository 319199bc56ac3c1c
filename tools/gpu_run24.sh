R=r24
python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}_ncu1.log 2>&1
python tools/summarize_ncu.py launches gpurun_out/${R}_launches.csv --last-eval | head -20
timeout 600 ncu --set full --clock-control none --import-source on -k regex:m2l_i8_kernel -s 1 -c 1 -o gpurun_out/${R}_i8 python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}_ncu2.log 2>&1
tail -2 gpurun_out/${R}_ncu2.log
