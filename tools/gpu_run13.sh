timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3 > gpurun_out/r13_pytest.log
cat gpurun_out/r13_pytest.log
timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats > gpurun_out/r13_stats.log 2>&1
grep -E "m2l|m2m|timings" gpurun_out/r13_stats.log
for c in 1 3 4; do
  timeout 600 python tools/run_config.py --cfg $c --evals 2 --stats > gpurun_out/r13_cfg$c.json 2> gpurun_out/r13_cfg$c.err
  echo "cfg$c rc=$?"; tail -2 gpurun_out/r13_cfg$c.err
done
