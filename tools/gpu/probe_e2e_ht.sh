cd $GRAFT_REPO_ROOT
F4B_HOST_TRACE=1 timeout 300 python tools/probe_e2e.py > gpurun_out/probe_e2e_ht.log 2>&1
echo done
