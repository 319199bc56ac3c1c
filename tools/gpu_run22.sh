R=r22
timeout 900 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -3 > gpurun_out/${R}_pytest.log
cat gpurun_out/${R}_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${R}_ref.json 2> gpurun_out/${R}_ref.err
cat gpurun_out/${R}_bench.json gpurun_out/${R}_ref.json
python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}_ncu1.log 2>&1
# full capture of the longest gather-GEMM launch of the timed eval
IDX=$(python - <<'EOF'
import csv
rows = [r for r in csv.reader(open("gpurun_out/r22_launches.csv")) if len(r) > 10]
hdr = rows[0]; k = hdr.index("Kernel Name"); v = hdr.index("Metric Value")
g = [float(r[v].replace(",", "")) for r in rows[1:] if "gather_gemm_tma" in r[k]]
half = len(g) // 2  # second eval (after warm-up)
i = max(range(half, len(g)), key=lambda j: g[j])
print(i)
EOF
)
echo "longest tma launch index $IDX"
ncu --set full --clock-control none --import-source on -k regex:gather_gemm_tma -s $IDX -c 1 -o gpurun_out/${R}_m2l python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}_ncu2.log 2>&1
tail -2 gpurun_out/${R}_ncu2.log
