cd $GRAFT_REPO_ROOT
for rb in 1 2 3 4 6; do
  echo "RB=$rb" >> gpurun_out/mr_rb.log
  F4B_SWEEP_RB=$rb timeout 300 python tools/probe_batches.py --brief --reps 2 --batches 10,19,27 2>&1 | grep batch >> gpurun_out/mr_rb.log
done
