R=r111
python tools/run_cfg2.py --warm 3 --evals 10 --stats > gpurun_out/${R}_base.log 2>&1
PKGPU_TRANS=i8 python tools/run_cfg2.py --warm 3 --evals 10 --stats > gpurun_out/${R}_tr.log 2>&1
for f in base tr; do python tools/stage_ms.py gpurun_out/${R}_$f.log 10 m2l pinv_up pinv_dn m2m l2l leaf tree lists s2m x periodic; done
PKGPU_TRANS=i8 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_tr.csv python tools/run_cfg2.py --warm 1 --evals 1 > /dev/null 2>&1
python tools/launch_times.py gpurun_out/${R}_tr.csv short | awk '{n=$NF; $NF=""; s[$0]+=n; c[$0]++} END {for (k in s) printf "%-45s %3d %.3f\n", k, c[k], s[k]}' | sort -k3 -nr | head -20
