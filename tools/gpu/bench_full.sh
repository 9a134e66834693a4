cd $GRAFT_REPO_ROOT
s=$(date +%s); timeout 1500 python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo bench rc=$? elapsed=$(( $(date +%s) - s ))s
