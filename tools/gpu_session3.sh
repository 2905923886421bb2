cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/pytest_kernels.log 2>&1; echo rc=$? >> gpurun_out/pytest_kernels.log
for s in video image cross_image; do
  for i in 4 5; do DF_ATTN_IMPL=$i timeout 120 python tools/attn_bench.py --shape $s; done
done > gpurun_out/attn_pair3.log 2>&1
timeout 300 python tools/profile_step.py --config image --steps 3 --kstats > gpurun_out/step_image.log 2>&1
DF_GEMM_SK=0 timeout 300 python tools/profile_step.py --config image --steps 3 --kstats >> gpurun_out/step_image.log 2>&1
DF_ATTN_IMPL=5 timeout 300 python tools/profile_step.py --config image --steps 3 --kstats >> gpurun_out/step_image.log 2>&1
