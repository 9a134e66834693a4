cd $GRAFT_REPO_ROOT
for i in 1 2; do
timeout 600 python bench.py --steps 10 --no-micro --no-cpu-baseline --no-systems --no-katsura11 --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
sp=d['symbolic_per_step']
print('AB', round(d['value']/1e9,4), d['kernels_top'].get('k_fbsp')['ms'], [sp[k]['t_us'] for k in ('0','3','5','8','10','19','27','30','36')])
"
done
