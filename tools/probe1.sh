set -x
nproc; lscpu | grep -E 'Model name|Socket|Core|Thread|MHz' ; free -g | head -2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/probe1_clocks.csv &
SMI=$!
./tools/fp64_peaks | tee gpurun_out/probe1_peaks.jsonl
kill $SMI
R=./oracle/_ref/refdump
mkdir -p /tmp/c2 && $R gen --n 100000 --kind uniform --ks 3 --out /tmp/c2/c2
export OMP_NUM_THREADS=$(nproc) OPENBLAS_NUM_THREADS=$(nproc)
timeout 300 $R eval --kernel stokeslet --per tp --ell 2 --p 8 --leaf 50 --src /tmp/c2/c2.src.f64 --str /tmp/c2/c2.str.f64 --op operators/stokeslet_tp_ell2_p8.pkm2l --repeat 2 | tee gpurun_out/probe1_ref_c2.json
