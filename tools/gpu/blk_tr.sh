cd $GRAFT_REPO_ROOT
F4B_BLK_TRACE=1 timeout 300 python tools/probe_batches.py --brief --reps 2 --batches 10,19,27 > gpurun_out/blk_tr.log 2>&1
F4B_DENSE_NOSR=1 F4B_BLK_TRACE=1 timeout 300 python tools/probe_batches.py --brief --reps 2 --batches 19 > gpurun_out/blk_tr2.log 2>&1
echo done
