cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/hostprep_test.log 2>&1; echo gputest rc=$?
F4B_HOST_TRACE=1 timeout 600 python tools/probe_batches.py --brief --reps 3 --batches 10,20,30,35 > gpurun_out/host_gap2.log 2>&1
timeout 600 python bench.py --steps 5 --no-micro --no-cpu-baseline --no-systems --no-katsura11 --e2e-steps 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('QB', d['value'], d['ms_per_step'], d['e2e']['value'], d['kernels_top'].get('k_dense_blk'), d['kernels_top'].get('k_fbsp'))
"
