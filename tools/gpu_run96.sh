R=r96
mkdir -p gpurun_out/${R}_ops
export LD_LIBRARY_PATH=/opt/prime-rl/.venv/lib/python3.12/site-packages/opencv_python_headless.libs:$LD_LIBRARY_PATH
for e in "madelung1d --p-list 6,8" "laplace-dp-pair --p-list 8" "stokes-tp-force --p-list 8" "stokes-tp-dipole --p-list 8,10"; do
  t0=$(date +%s.%N); timeout 900 ./oracle/_ref/pkifmm_dropin $e --operator-dir gpurun_out/${R}_ops >> gpurun_out/${R}_dropin.jsonl 2>> gpurun_out/${R}_dropin.err; rc=$?; echo "rc=$rc $e seconds=$(echo "$(date +%s.%N) - $t0" | bc)" >> gpurun_out/${R}_dropin.jsonl
done
cat gpurun_out/${R}_dropin.jsonl; tail -8 gpurun_out/${R}_dropin.err
