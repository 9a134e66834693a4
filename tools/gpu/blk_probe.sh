cd $GRAFT_REPO_ROOT
F4B_BLK_TRACE=1 python tools/probe_batches.py --brief --reps 2 --batches 7,10,17,19,27 > gpurun_out/blk_probe.log 2>&1; echo probe rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-micro --no-cpu-baseline --e2e-steps 0 --no-katsura11 > gpurun_out/bench_blk.log 2>&1; echo bench rc=$?
