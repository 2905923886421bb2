cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attn_sk.py tests/test_gpu_kernels.py -q -x -k "attn or attention" > gpurun_out/sk_test.log 2>&1; echo rc=$? >> gpurun_out/sk_test.log
for s in cross_image cross_video; do timeout 120 python tools/attn_bench.py --shape $s --reps 20 --iters 5 >> gpurun_out/sk_bench.log 2>&1; DF_ATTN_SK=0 timeout 120 python tools/attn_bench.py --shape $s --reps 20 --iters 5 >> gpurun_out/sk_bench.log 2>&1; done
