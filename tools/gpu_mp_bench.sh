# The N > 1 bench path exercised on one GPU (two processes on device 0, gloo plumbing), plus
# the newest multi-process and FP8 tests.  Run under gpurun from the repo root.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_fp8.py -q --durations=5 > gpurun_out/pytest_mp_fp8.log 2>&1; echo rc=$? >> gpurun_out/pytest_mp_fp8.log
DF_BENCH_DEVICE=0 DF_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_2proc.json 2> gpurun_out/bench_2proc.err
