R=r93
for M in 1 9 65; do PKGPU_M2L_I8_MIN=$M timeout 300 python tools/run_cfg2.py --evals 6 --warm 2 --stats > gpurun_out/${R}_m$M.log 2>&1; echo "min=$M $(grep -E '^timings' gpurun_out/${R}_m$M.log | cut -c1-80) $(python - gpurun_out/${R}_m$M.log <<'P'
import sys,ast
d={}
for line in open(sys.argv[1]):
    k,_,v=line.partition(' ')
    if k in ('m2l','m2l_i8'): d[k]=round(ast.literal_eval(v)['seconds']/6*1e3,3)
print(d)
P
)"; done
