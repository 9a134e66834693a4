cd $GRAFT_REPO_ROOT
timeout 600 python tools/micro/mb_dict.py 5 > gpurun_out/micro_bench.log 2>&1; echo rc=$? >> gpurun_out/micro_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"msd|mb_|sort|scan|k_" --csv --log-file gpurun_out/micro_ncu.csv python tools/micro/mb_dict.py 1 > gpurun_out/micro_ncu.log 2>&1; echo ncu rc=$? >> gpurun_out/micro_bench.log
