cd $GRAFT_REPO_ROOT
F4B_BLK_TRACE=1 timeout 600 python tools/probe_batches.py --brief --reps 2 --batches 10,17,19,27 > gpurun_out/blk_probe3.log 2>&1; echo probe rc=$?
