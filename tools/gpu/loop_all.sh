cd $GRAFT_REPO_ROOT
F4B_LOOP_TRACE=1 timeout 600 python tools/probe_batches.py --brief --reps 2 --batches $(python -c "print(','.join(str(i) for i in range(38)))") > gpurun_out/loop_all.log 2>&1; echo rc=$?
