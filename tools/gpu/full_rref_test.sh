cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "psge or full_rref or large_step_replay or full_run" > gpurun_out/frr_test.log 2>&1; echo parity rc=$?
timeout 300 python bench.py --steps 5 --no-micro --no-cpu-baseline --no-katsura11 --no-systems --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('QB', d['value'], d['ms_per_step'], d['reduction_full_rref']['s_per_f4_step'])
"
