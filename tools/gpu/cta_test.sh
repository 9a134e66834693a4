cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -x -q -k "compile or f4_steps or large_step_replay or full_run or katsura11 or shard or wiedemann" > gpurun_out/cta_test.log 2>&1; echo parity rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-micro --no-cpu-baseline --e2e-steps 1 --no-katsura11 > gpurun_out/bench_cta.log 2>&1; echo bench rc=$?
