cd $GRAFT_REPO_ROOT
for g in 0 148 74; do
  F4B_PREP_G=$g timeout 300 python bench.py --steps 5 --no-micro --no-cpu-baseline --no-katsura11 --no-systems --e2e-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('G=$g', d['value'], d['ms_per_step'], d['kernels_top'].get('k_psge_prep'))
"
done
