#!/bin/bash
# One parameterised GPU-box runner (run under gpurun from the repo root):
#   bash tools/gpu_run.sh TAG STEP [STEP ...]
# Steps: smi | pytest | pytest:<-k expr> | smoke | bench | bench:<args> | launches | cfg<N> |
#        ncu:<kernel regex> | sanitize:<tool>
# Outputs go to gpurun_out/TAG_*. Per-call experiment scripts live in tools/scratch/ (git-ignored).
TAG=$1; shift
O=gpurun_out/${TAG}
mkdir -p gpurun_out
for S in "$@"; do
  case "$S" in
    smi) nvidia-smi > ${O}_smi.txt; lscpu > ${O}_lscpu.txt ;;
    pytest) timeout 1800 python -m pytest tests -m gpu -x -q > ${O}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 ${O}_pytest.log ;;
    pytest:*) timeout 1800 python -m pytest tests -m gpu -x -q -s -k "${S#pytest:}" > ${O}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 ${O}_pytest.log ;;
    smoke) timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 ${O}_smoke.log ;;
    bench) timeout 900 python bench.py > ${O}_bench.json 2> ${O}_bench.err; echo "bench rc=$?" ;;
    bench:*) timeout 900 python bench.py ${S#bench:} > ${O}_bench.json 2> ${O}_bench.err; echo "bench rc=$?" ;;
    launches) timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
                --log-file ${O}_launches.csv python tools/run_cfg2.py --warm 1 --evals 1 > /dev/null 2>&1; echo "launches rc=$?" ;;
    cfg*) C=${S#cfg}; timeout 1500 python tools/run_config.py --cfg $C --evals $([ $C = 5 ] && echo 1 || echo 5) --stats \
                > ${O}_cfg$C.json 2> ${O}_cfg$C.err; echo "cfg$C rc=$? $(grep -o '"ms_per_eval": [0-9.]*' ${O}_cfg$C.json)" ;;
    ncu:*) timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:${S#ncu:}" -c 1 \
                -o ${O}_$(echo ${S#ncu:} | tr -c 'a-zA-Z0-9_\n' _) python tools/run_cfg2.py --warm 1 --evals 1 > ${O}_ncu.log 2>&1; echo "ncu rc=$?" ;;
    sanitize:*) timeout 1500 compute-sanitizer --tool ${S#sanitize:} --error-exitcode 9 python -m pytest -x -q -p no:cacheprovider \
                tests/test_gpu_i8.py::test_i8_gather_gemm_exact "tests/test_gpu_parity.py::test_evaluate_vs_reference[lap_sp_p8_clu]" \
                > ${O}_sanitize_${S#sanitize:}.log 2>&1; echo "sanitize ${S#sanitize:} rc=$?"; tail -3 ${O}_sanitize_${S#sanitize:}.log ;;
    *) bash "$S" ;;
  esac
done
