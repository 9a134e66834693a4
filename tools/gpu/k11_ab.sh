cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tab_test.log 2>&1; echo gputest rc=$?
timeout 900 python bench.py --steps 5 --no-micro --no-cpu-baseline --no-systems --e2e-steps 2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
k=d['katsura11']
print('AB', round(d['value']/1e9,4), d['e2e']['value'], k['wall_s'], {s:v['t_sym_us'] for s,v in k['warm_replays'].items()})
"
