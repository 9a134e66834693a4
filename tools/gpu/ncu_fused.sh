cd $GRAFT_REPO_ROOT
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k "regex:k_fused" -c 1 -o gpurun_out/fused_s19 \
  python tools/probe_batches.py --batches 19 --reps 1 --profile-region > gpurun_out/ncu_fused.log 2>&1; echo ncu rc=$?
