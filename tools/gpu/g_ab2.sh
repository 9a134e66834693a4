cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gab_test.log 2>&1; echo gputest rc=$?
for env in "" "F4B_FBSP_G=296" "" "F4B_FBSP_G=296"; do
env $env timeout 600 python bench.py --steps 10 --no-micro --no-cpu-baseline --no-systems --no-katsura11 --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
sp=d['symbolic_per_step']
print('AB [$env]', d['value'], d['kernels_top'].get('k_fbsp'), [sp[k]['t_us'] for k in ('0','3','5','8','10','19','27','30','36')])
"
done
