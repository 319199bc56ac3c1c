for c in 1 3 4; do
  timeout 600 python tools/run_config.py --cfg $c --evals 2 --stats > gpurun_out/r12_cfg$c.json 2> gpurun_out/r12_cfg$c.err
  echo "cfg$c rc=$?"; tail -2 gpurun_out/r12_cfg$c.err
done
timeout 900 python tools/run_config.py --cfg 5 --evals 1 --stats > gpurun_out/r12_cfg5.json 2> gpurun_out/r12_cfg5.err
echo "cfg5 rc=$?"; tail -2 gpurun_out/r12_cfg5.err
cat gpurun_out/r12_cfg*.json | cut -c1-400
