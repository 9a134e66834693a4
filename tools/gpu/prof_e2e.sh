cd $GRAFT_REPO_ROOT
timeout 600 python tools/prof_e2e.py > gpurun_out/prof_e2e.log 2>&1; echo rc=$?
