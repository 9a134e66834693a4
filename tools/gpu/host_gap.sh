cd $GRAFT_REPO_ROOT
F4B_HOST_TRACE=1 timeout 600 python tools/probe_batches.py --brief --reps 3 --batches $(python -c "print(','.join(map(str,range(38))))") > gpurun_out/host_gap.log 2>&1
echo rc=$?
