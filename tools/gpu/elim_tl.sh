cd $GRAFT_REPO_ROOT
F4B_ELIM_TRACE=0 timeout 600 python tools/probe_batches.py --brief --reps 2 --batches 3,10,19,27,33 > gpurun_out/elim_tl.log 2>&1; echo probe rc=$?
