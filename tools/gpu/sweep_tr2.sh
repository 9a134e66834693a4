cd $GRAFT_REPO_ROOT
bash tools/gpu/sweep_tr.sh
timeout 600 python bench.py --steps 5 --warmup 3 --no-micro --no-cpu-baseline --e2e-steps 0 --no-katsura11 > gpurun_out/bench_sweep.log 2>&1; echo bench rc=$?
