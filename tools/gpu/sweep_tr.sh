cd $GRAFT_REPO_ROOT
F4B_SWEEP_TRACE=1 timeout 600 python tools/probe_batches.py --brief --reps 1 --batches 10,17,19,21,27,33 > gpurun_out/sweep_tr.log 2>&1; echo probe rc=$?
