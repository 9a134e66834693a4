cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f4host_test.log 2>&1; echo gputest rc=$?
timeout 600 python tools/prof_f4.py cyclic 8 > gpurun_out/prof_f4.log 2>&1; echo prof rc=$?
timeout 900 python bench.py --steps 5 --no-micro --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('QB', d['value'], d['ms_per_step'], d['e2e']['value'], d['setup_s'], d['full_run'], d['katsura11'].get('wall_s') if d['katsura11'] else None)
print('SYS', json.dumps(d['other_systems'])[:1500])
print('K11', json.dumps(d['katsura11'])[:1500])
"
