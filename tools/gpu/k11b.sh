cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/k11b_test.log 2>&1; echo gputest rc=$?
timeout 600 python tools/prof_f4.py katsura 11 > gpurun_out/prof_k11.log 2>&1; echo prof rc=$?
timeout 600 python tools/prof_f4.py cyclic 8 > gpurun_out/prof_f4.log 2>&1; echo prof rc=$?
