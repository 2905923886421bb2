cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attn_sk.py tests/test_gpu_kernels.py -q -x -k "attn or attention or short" > gpurun_out/sk4_test.log 2>&1; echo rc=$? >> gpurun_out/sk4_test.log
timeout 900 python bench.py --config video --precision mxfp8 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_video_mxfp8.json 2> gpurun_out/bench_video_mxfp8.err
