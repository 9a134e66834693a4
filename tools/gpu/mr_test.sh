cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "psge or large_step_replay or f4_steps or full_run" > gpurun_out/mr_test.log 2>&1; echo parity rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-micro --no-cpu-baseline --e2e-steps 0 --no-katsura11 > gpurun_out/bench_mr.log 2>&1; echo bench rc=$?
timeout 300 python tools/probe_batches.py --brief --reps 2 --batches 10,17,19,27 > gpurun_out/mr_probe.log 2>&1
