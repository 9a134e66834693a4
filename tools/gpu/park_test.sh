cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -k "not fallback_paths" > gpurun_out/park_test.log 2>&1; echo gputest rc=$?
timeout 900 python bench.py --steps 5 --no-micro --no-cpu-baseline --no-systems --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('QB', d['value'], d['ms_per_step'], d['kernels_top'].get('k_fbsp'), {k: v['t_sym_us'] for k, v in d['katsura11']['warm_replays'].items()})
"
