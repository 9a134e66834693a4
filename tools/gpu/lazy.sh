cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/lazy_test.log 2>&1; echo gputest rc=$?
F4B_HOST_TRACE=1 timeout 300 python tools/probe_e2e.py > gpurun_out/probe_e2e_ht.log 2>&1
timeout 600 python bench.py --steps 5 --no-micro --no-cpu-baseline --no-systems --no-katsura11 --e2e-steps 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('QB', d['value'], d['ms_per_step'], d['e2e']['value'])
"
