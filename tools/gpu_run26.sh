R=r26
./tools/i8_peak > gpurun_out/${R}_i8peak.json 2>&1; cat gpurun_out/${R}_i8peak.json
timeout 900 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -4 > gpurun_out/${R}_pytest.log
cat gpurun_out/${R}_pytest.log
timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats > gpurun_out/${R}_stats.log 2>&1
grep -E "^m2l|timings|Error|error" gpurun_out/${R}_stats.log
python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}_ncu1.log 2>&1
python tools/summarize_ncu.py launches gpurun_out/${R}_launches.csv --last-eval > gpurun_out/${R}_launches.md 2>&1; head -14 gpurun_out/${R}_launches.md
IDX=$(python - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/r26_launches.csv")) if len(r) > 10]
hdr = rows[0]; k = hdr.index("Kernel Name"); v = hdr.index("Metric Value")
g = [float(r[v].replace(",", "")) for r in rows[1:] if "m2l_i8_kernel" in r[k]]
half = len(g) // 2
print(max(range(half, len(g)), key=lambda j: g[j]))
PY
)
echo "longest i8 launch index $IDX"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:m2l_i8_kernel -s $IDX -c 1 -o gpurun_out/${R}_i8 python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}_ncu2.log 2>&1
tail -1 gpurun_out/${R}_ncu2.log
timeout 1500 python tools/quant_study.py --specs "dmma;i8all:17,56,56;i8all:16,53,53;i8all:16,52,52;i8all:15,49,49;i8all:14,45,45" > gpurun_out/${R}_quant.jsonl 2>&1
cut -c1-200 gpurun_out/${R}_quant.jsonl
