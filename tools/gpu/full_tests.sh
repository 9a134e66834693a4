cd $GRAFT_REPO_ROOT
timeout 3000 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gputest_full.log 2>&1; echo gputest rc=$?
