cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "stream_k or integer" > gpurun_out/pytest_sk.log 2>&1
for tc in 1 2; do timeout 120 python tools/gemm_bench.py --no-cublas --tc $tc --only image_o; timeout 120 python tools/gemm_bench.py --no-cublas --tc $tc --only image_down; done > gpurun_out/gemm_sk.log 2>&1
for s in video image; do DF_ATTN_IMPL=5 timeout 120 python tools/attn_bench.py --shape $s | sed "s/^/pair3q /"; done >> gpurun_out/gemm_sk.log 2>&1
timeout 300 python tools/profile_step.py --config image --steps 4 --kstats > gpurun_out/step_image.log 2>&1
DF_GEMM_SK=1 timeout 300 python tools/profile_step.py --config image --steps 4 --kstats >> gpurun_out/step_image.log 2>&1
