cd $GRAFT_REPO_ROOT
for env in "" "F4B_NO_PREFETCH=1"; do
env $env timeout 900 python bench.py --steps 3 --no-micro --no-cpu-baseline --no-systems --e2e-steps 2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
k=d['katsura11']
print('AB [$env]', d['value'], d['e2e']['value'], k['wall_s'], {s:(v['t_sym_us'], v['first_touch_us']) for s,v in k['warm_replays'].items()}, k['live_sym_ms_per_step'])
"
done
