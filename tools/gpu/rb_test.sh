cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "full_run or reduce_basis or katsura11 or f4_groebner or snapshot" > gpurun_out/rb_test.log 2>&1; echo parity rc=$?
timeout 600 python tools/full_run.py katsura 12 --max-steps 30 > gpurun_out/k12_full.log 2>&1; echo k12 rc=$?
timeout 300 python tools/full_run.py katsura 11 > gpurun_out/k11_full.log 2>&1; echo k11 rc=$?
