cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "psge or large_step_replay or f4_steps or full_run or katsura" > gpurun_out/ps_test.log 2>&1; echo parity rc=$?
F4B_BLK_TRACE=1 timeout 300 python tools/probe_batches.py --brief --reps 2 --batches 10,19,27 > gpurun_out/ps_tr.log 2>&1
timeout 300 python bench.py --steps 5 --no-micro --no-cpu-baseline --no-katsura11 --no-systems --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('QB', d['value'], d['ms_per_step'], d['kernels_top'].get('k_dense_blk'))
"
