cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_shard.py -x -q > gpurun_out/shard_test.log 2>&1; echo shard rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q -k "not fallback_paths and not shard" > gpurun_out/gputest_quick.log 2>&1; echo gputest rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-micro --no-cpu-baseline --e2e-steps 0 --no-katsura11 > gpurun_out/bench_quick.log 2>&1; echo bench rc=$?
F4B_LOOP_TRACE=1 F4B_HOST_TRACE=1 python tools/probe_batches.py --brief --reps 3 --batches 0,5,10,19 > gpurun_out/probe_fbsp2.log 2>&1
