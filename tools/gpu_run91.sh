R=r91
for U in 8 16 32 64; do PKGPU_GEMM_UNITS=$U timeout 300 python tools/run_cfg2.py --evals 6 --warm 2 --stats > gpurun_out/${R}_u$U.log 2>&1; echo "units=$U $(python - gpurun_out/${R}_u$U.log <<'P'
import sys,ast
d={}
for line in open(sys.argv[1]):
    k,_,v=line.partition(' ')
    if k in ('m2m','l2l','pinv_up','pinv_dn'): d[k]=round(ast.literal_eval(v)['seconds']/6*1e3,3)
print(d, round(sum(d.values()),3))
P
)"; done
