cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tab_test.log 2>&1; echo gputest rc=$?
bash tools/gpu/ab_simple.sh
