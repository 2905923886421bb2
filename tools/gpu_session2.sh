cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_scheduler.py -x -q > gpurun_out/pytest_pipe.log 2>&1; echo rc=$? >> gpurun_out/pytest_pipe.log
for s in video image; do
  for i in 2 4; do DF_ATTN_IMPL=$i timeout 120 python tools/attn_bench.py --shape $s; done
  DF_ATTN_IMPL=4 DF_ATTN_POLY=1 timeout 120 python tools/attn_bench.py --shape $s | sed 's/^/poly /'
done > gpurun_out/attn_tc3.log 2>&1
DF_ATTN_IMPL=4 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "bruteforce or special_cases" > gpurun_out/pytest_attn4.log 2>&1
timeout 300 python tools/profile_step.py --config image --steps 3 --kstats > gpurun_out/step_image.log 2>&1
DF_ATTN_IMPL=4 timeout 300 python tools/profile_step.py --config image --steps 3 --kstats >> gpurun_out/step_image.log 2>&1
