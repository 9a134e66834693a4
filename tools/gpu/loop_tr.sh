cd $GRAFT_REPO_ROOT
F4B_LOOP_TRACE=1 timeout 300 python tools/probe_batches.py --brief --reps 2 --batches 0,3,11,29,33,19 > gpurun_out/loop_tr.log 2>&1; echo rc=$?
