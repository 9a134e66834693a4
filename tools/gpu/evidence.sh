cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ev
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err; echo ref rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/ev/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-micro --no-katsura11 --no-systems --e2e-steps 0 --no-cpu-baseline > gpurun_out/ev/ncu_bench.log 2>&1; echo ncu rc=$?
python tools/probe_batches.py --batches 19 --reps 2 > gpurun_out/ev/probe_s19_plain.log 2>&1; echo plain rc=$?
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k "regex:k_fbsp|k_sweep_win|k_dense_blk|k_win_build|k_psge_prep|k_tail_copy" -c 6 -o gpurun_out/ev/full_s19_r02 \
  python tools/probe_batches.py --batches 19 --reps 1 --profile-region > gpurun_out/ev/ncu_s19.log 2>&1; echo ncu_full rc=$?
