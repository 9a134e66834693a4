cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 5 --no-micro --no-cpu-baseline --no-katsura11 --no-systems --e2e-steps 0 > gpurun_out/qb.log 2>&1; echo bench rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/qb.log').readlines()[-1]); print('QB', d['value'], d['ms_per_step'], list(d['kernels_top'].items())[:5])"
