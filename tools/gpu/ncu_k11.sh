cd $GRAFT_REPO_ROOT
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:k_fbsp" -c 1 \
  -o gpurun_out/k11_s8_fbsp python tools/full_run.py katsura 11 --max-steps 9 --profile-step 8 > gpurun_out/ncu_k11.log 2>&1; echo rc=$?
