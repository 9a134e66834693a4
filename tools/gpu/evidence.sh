cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ev
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err; echo ref rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/ev/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-micro --no-katsura11 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ev/ncu_bench.log 2>&1; echo ncu rc=$?
