timeout 900 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -3 > gpurun_out/r16_pytest.log
cat gpurun_out/r16_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r16_bench.json 2> gpurun_out/r16_bench.err
python -c "import json;d=json.load(open('gpurun_out/r16_bench.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac'])"
tail -3 gpurun_out/r16_bench.err
