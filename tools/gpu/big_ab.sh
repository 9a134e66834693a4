cd $GRAFT_REPO_ROOT
for env in "F4B_FBSP_BIG_NF=0" "F4B_FBSP_BIG_NF=600" "F4B_FBSP_BIG_NF=1200" "F4B_FBSP_BIG_NF=4800" "F4B_FBSP_BIG_NF=100000" "F4B_FBSP_BIG_NF=0" "F4B_FBSP_BIG_NF=1200" "F4B_FBSP_BIG_NF=4800"; do
env $env timeout 600 python bench.py --steps 10 --no-micro --no-cpu-baseline --no-systems --no-katsura11 --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
sp=d['symbolic_per_step']
print('AB [$env]', round(d['value']/1e9,4), d['kernels_top'].get('k_fbsp')['ms'], [sp[k]['t_us'] for k in ('0','3','5','8','10','19','27','30','36')])
"
done
