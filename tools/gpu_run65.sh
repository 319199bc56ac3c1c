R=r65
timeout 400 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; tail -c 400 gpurun_out/${R}_bench.json
# ncu full captures of the two int8 M2L launches of a profiled evaluate (small-level run, level 4)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:m2l_i8 --launch-skip 2 --launch-count 2 -o gpurun_out/${R}_m2l python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pkgpu --launch-skip 0 --csv --log-file gpurun_out/${R}_launches.csv python tools/run_cfg2.py --evals 1 --warm 0 > /dev/null 2>&1
ls gpurun_out | grep $R
