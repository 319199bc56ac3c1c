R=r78
for C in 2 3 4; do timeout 900 python tools/run_config.py --cfg $C --evals 1 --stats > gpurun_out/${R}_cfg$C.json 2> gpurun_out/${R}_cfg$C.err; python -c "
import json; d=json.loads(open('gpurun_out/${R}_cfg$C.json').read().strip().splitlines()[-1]); st=d['stages']
print($C, d['ms_per_eval'], 'apps', st['m2l_i8']['units'], 'mma rows', st.get('m2l_mma_rows',{}).get('units'), 'ratio', st.get('m2l_mma_rows',{}).get('units',0)/max(1,st['m2l_i8']['units']))"; done
