R=r43
run() { timeout 300 python tools/run_cfg2.py --evals 6 --warm 2 --stats > gpurun_out/${R}_$1.log 2>&1; echo "$1 $(grep -E '^m2l_i8 ' gpurun_out/${R}_$1.log | cut -c1-48) $(grep -E '^m2l ' gpurun_out/${R}_$1.log | cut -c1-40)"; }
for P in 0 2 3; do for S in 1024 0; do PKGPU_I8_PAIR=$P PKGPU_I8_SMALL=$S run p${P}_s$S; done; done
PKGPU_I8_PAIR=1 PKGPU_I8_SMALL=0 run p1_s0
# per-launch list of the base config
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:m2l_i8 --csv --log-file gpurun_out/${R}_launches.csv python tools/run_cfg2.py --evals 1 --warm 1 > /dev/null 2>&1
PKGPU_I8_SMALL=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:m2l_i8 --csv --log-file gpurun_out/${R}_launches_s0.csv python tools/run_cfg2.py --evals 1 --warm 1 > /dev/null 2>&1
grep -c m2l gpurun_out/${R}_launches.csv
