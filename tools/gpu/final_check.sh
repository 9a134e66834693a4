cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_test.log 2>&1; echo gputest rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
for i in 1 2; do
timeout 600 python bench.py --steps 10 --no-micro --no-cpu-baseline --no-systems --e2e-steps 2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1])
print('QB', round(d['value']/1e9,4), d['ms_per_step'], d['e2e']['value'], d['kernels_top'].get('k_fbsp')['ms'], d['katsura11']['wall_s'], {s:v['t_sym_us'] for s,v in d['katsura11']['warm_replays'].items()})
"
done
