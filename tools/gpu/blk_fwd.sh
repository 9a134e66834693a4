cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/blk_fwd_test.log 2>&1; echo gputest rc=$?
F4B_BLK_TRACE=1 timeout 300 python tools/probe_batches.py --brief --reps 2 --batches 10,19,27 > gpurun_out/blk_tr3.log 2>&1
timeout 600 python bench.py --steps 5 --no-micro --no-cpu-baseline --no-systems --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('QB', d['value'], d['ms_per_step'], d['reduction_s_per_f4_step'], d['reduction_full_rref']['s_per_f4_step'], d['kernels_top'].get('k_dense_blk'), d['kernels_top'].get('k_fbsp'))
"
