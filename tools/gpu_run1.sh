set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -rA --timeout 600 2>&1 | tail -80 > gpurun_out/r1_pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err
tail -5 gpurun_out/r1_bench.err
cat gpurun_out/r1_bench.json
