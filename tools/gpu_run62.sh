R=r62
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_all.csv python tools/run_cfg2.py --evals 1 --warm 1 > /dev/null 2>&1
python tools/launch_times.py gpurun_out/${R}_all.csv x | awk '{n[$1]+=1; t[$1]+=$NF} END {for (k in n) printf "%-40s %5d %8.3f\n", k, n[k], t[k]}' | sort -k3 -n -r | head -30
