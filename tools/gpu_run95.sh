R=r95
for M in 16 8 4 2; do PKGPU_GEMM_MINIT=$M timeout 300 python tools/run_cfg2.py --evals 6 --warm 2 --stats > gpurun_out/${R}_m$M.log 2>&1; echo "minit=$M $(python - gpurun_out/${R}_m$M.log <<'P'
import sys,ast
d={}
for line in open(sys.argv[1]):
    k,_,v=line.partition(' ')
    if k in ('m2m','l2l','pinv_up','pinv_dn'): d[k]=round(ast.literal_eval(v)['seconds']/6*1e3,3)
print(d, round(sum(d.values()),3))
P
)"; done
