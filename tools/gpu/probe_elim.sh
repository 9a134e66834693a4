cd $GRAFT_REPO_ROOT
F4B_ELIM_TRACE=1 F4B_BLK_TRACE=1 python tools/probe_batches.py --reps 3 --batches 0,3,7,10,12,19,21,27 > gpurun_out/probe_elim.log 2>&1
echo probe rc=$?
