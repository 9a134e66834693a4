cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "prefetch or plan_text or validate" > gpurun_out/pf_test.log 2>&1; echo parity rc=$?
timeout 900 python bench.py --steps 5 --no-micro --no-cpu-baseline --no-katsura11 --no-systems --e2e-steps 2 > gpurun_out/bench_pf.log 2>&1; echo bench rc=$?
