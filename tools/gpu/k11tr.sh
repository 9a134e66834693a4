cd $GRAFT_REPO_ROOT
F4B_ELIM_TRACE=8 F4B_BLK_TRACE=1 timeout 600 python tools/full_run.py katsura 11 > gpurun_out/k11_tr.log 2>&1; echo k11 rc=$?
