cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "compile or f4_steps or large_step_replay or full_run or katsura11" > gpurun_out/fused_test.log 2>&1; echo parity rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-micro --no-cpu-baseline --e2e-steps 0 --no-katsura11 > gpurun_out/bench_fused.log 2>&1; echo bench rc=$?
F4B_LOOP_TRACE=1 python tools/probe_batches.py --brief --reps 3 --batches 0,5,10,19 > gpurun_out/probe_fused.log 2>&1
