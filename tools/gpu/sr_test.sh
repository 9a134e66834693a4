cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "psge or large_step_replay or f4_steps or full_run or katsura" > gpurun_out/sr_test.log 2>&1; echo parity rc=$?
for v in 0 1; do
  if [ $v = 1 ]; then export F4B_DENSE_NOSR=1; fi
  timeout 300 python bench.py --steps 5 --no-micro --no-cpu-baseline --no-katsura11 --no-systems --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('NOSR=$v', d['value'], d['ms_per_step'], d['kernels_top'].get('k_dense_blk'))
"
done
