cd $GRAFT_REPO_ROOT
F4B_BLK_TRACE=1 python tools/probe_batches.py --brief --reps 1 --batches 7,10,17,19,27 > gpurun_out/blk_probe2.log 2>&1; echo probe rc=$?
