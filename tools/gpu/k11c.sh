cd $GRAFT_REPO_ROOT
timeout 600 python tools/full_run.py katsura 11 > gpurun_out/k11_full.log 2>&1; echo k11 rc=$?
timeout 600 python tools/full_run.py katsura 11 > gpurun_out/k11_full2.log 2>&1; echo k11 rc=$?
