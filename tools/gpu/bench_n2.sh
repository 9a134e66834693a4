cd $GRAFT_REPO_ROOT
F4B_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 2 --warmup 3 --no-micro --no-katsura11 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_n2.log 2>&1; echo n2 rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "f4_steps or wiedemann or snapshot" > gpurun_out/t_dev.log 2>&1; echo tests rc=$?
