cd $GRAFT_REPO_ROOT
timeout 300 python tools/micro/mb_dict.py 1 > gpurun_out/mbfull_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_msd_bucket" --launch-skip 0 --launch-count 1 -o gpurun_out/msd_bucket50 python tools/micro/mb_dict.py 1 > gpurun_out/mbfull_ncu.log 2>&1; echo ncu rc=$?
