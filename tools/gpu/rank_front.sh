cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "compile or f4_steps or large_step_replay or full_run or katsura11 or wiedemann or plan_text" > gpurun_out/rf_test.log 2>&1; echo parity rc=$?
timeout 900 python bench.py --steps 5 --warmup 3 --no-micro --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_rf.log 2>&1; echo bench rc=$?
F4B_LOOP_TRACE=1 python tools/full_run.py katsura 11 > gpurun_out/k11_trace2.log 2>&1
