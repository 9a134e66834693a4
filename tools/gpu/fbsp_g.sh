cd $GRAFT_REPO_ROOT
for g in 0 16 32 64 148; do
  echo "G=$g" >> gpurun_out/fbsp_g.log
  F4B_FBSP_G=$g timeout 300 python bench.py --steps 3 --no-micro --no-cpu-baseline --no-katsura11 --no-systems --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'])
print('per', {k: v['t_us'] for k, v in d['symbolic_per_step'].items()})
" >> gpurun_out/fbsp_g.log 2>&1
done
