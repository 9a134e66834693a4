cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_micro.py -q -x > gpurun_out/micro_test.log 2>&1; echo micro rc=$? >> gpurun_out/micro_test.log
timeout 600 python - > gpurun_out/micro_bench.log 2>&1 <<'P'
import json
from paper_2601_06765_b200.bench import microbench
for dup in (0.5, 0.99, 0.0):
    d = microbench("dict_build", 1 << 24, duplicate_rate=dup, seed=1, reps=5)
    print(json.dumps({k: d[k] for k in ("duplicate_rate", "unique_out", "elapsed_ns", "hbm_frac", "hbm_frac_streamed", "dict_path")}))
P
echo bench rc=$? >> gpurun_out/micro_bench.log
