cd $GRAFT_REPO_ROOT
for v in 0 1 2 3 4; do
  echo "== SWV=$v" >> gpurun_out/swv.log
  F4B_SWV=$v timeout 300 python tools/probe_batches.py --brief --reps 3 --batches 10,19,21,27 >> gpurun_out/swv.log 2>&1
  F4B_SWV=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-micro --no-cpu-baseline --e2e-steps 0 --no-katsura11 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('bench', d['ms_per_step'], [(k, v) for k, v in d.get('kernels_top', {}).items()][:4])" >> gpurun_out/swv.log 2>&1
done
