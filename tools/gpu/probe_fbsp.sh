cd $GRAFT_REPO_ROOT
F4B_LOOP_TRACE=1 F4B_HOST_TRACE=1 python tools/probe_batches.py --brief --reps 3 --batches 0,3,5,7,10,19,21 > gpurun_out/probe_fbsp.log 2>&1
echo probe rc=$?
timeout 3000 python -m pytest tests -m gpu -x -q --durations=30 > gpurun_out/gputest.log 2>&1; echo gputest rc=$?
