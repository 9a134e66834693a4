cd $GRAFT_REPO_ROOT
python tools/probe_batches.py --batches 19 --reps 2 > gpurun_out/probe_s19_plain.log 2>&1; echo plain rc=$?
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k "regex:k_fbsp|k_sweep_win|k_dense_blk|k_win_build|k_psge_prep" -c 5 -o gpurun_out/full_s19_r02 \
  python tools/probe_batches.py --batches 19 --reps 1 --profile-region > gpurun_out/ncu_s19.log 2>&1; echo ncu rc=$?
