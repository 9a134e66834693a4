cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/red6_test.log 2>&1; echo gputest rc=$?
for i in 1 2; do
timeout 600 python bench.py --steps 10 --no-micro --no-cpu-baseline --no-systems --no-katsura11 --e2e-steps 2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('QB', d['value'], d['ms_per_step'], d['e2e']['value'], d['kernels_top'].get('k_fbsp'))
"
done
