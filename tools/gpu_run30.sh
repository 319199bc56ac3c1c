R=r30
export PKGPU_I8_PAIR=1
python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}_ncu1.log 2>&1
python tools/summarize_ncu.py launches gpurun_out/${R}_launches.csv --last-eval > gpurun_out/${R}_launches.md 2>&1; head -8 gpurun_out/${R}_launches.md
grep m2l_i8 gpurun_out/${R}_launches.csv | tail -4 | cut -c1-300
IDX=$(python - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/r30_launches.csv")) if len(r) > 10]
hdr = rows[0]; k = hdr.index("Kernel Name"); v = hdr.index("Metric Value")
g = [float(r[v].replace(",", "")) for r in rows[1:] if "m2l_i8" in r[k]]
half = len(g) // 2
print(max(range(half, len(g)), key=lambda j: g[j]))
PY
)
echo "longest i8 launch index $IDX"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:m2l_i8 -s $IDX -c 1 -o gpurun_out/${R}_pair python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}_ncu2.log 2>&1
tail -1 gpurun_out/${R}_ncu2.log
