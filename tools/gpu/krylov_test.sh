cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "resident_operator or left_kernel or wiedemann or syzygy or bm" > gpurun_out/krylov_test.log 2>&1; echo parity rc=$?
timeout 600 python bench.py --steps 3 --no-micro --no-cpu-baseline --no-katsura11 --e2e-steps 0 > gpurun_out/bench_sys.log 2>&1; echo bench rc=$?
