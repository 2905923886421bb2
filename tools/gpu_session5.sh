cd $GRAFT_REPO_ROOT
for tc in 1 2; do DF_GEMM_VERBOSE=1 timeout 120 python tools/gemm_bench.py --no-cublas --tc $tc --only image_o; timeout 120 python tools/gemm_bench.py --no-cublas --tc $tc --only image_down; done > gpurun_out/gemm_sk.log 2>&1
for s in video image; do
  for m in 0 2 3; do DF_ATTN_IMPL=4 DF_ATTN_POLY=$m timeout 120 python tools/attn_bench.py --shape $s | sed "s/^/tc3 m$m /"; done
  for m in 0 2 3; do DF_ATTN_IMPL=5 DF_ATTN_POLY=$m timeout 120 python tools/attn_bench.py --shape $s | sed "s/^/pair3 m$m /"; done
done > gpurun_out/attn_modes.log 2>&1
timeout 300 python tools/profile_step.py --config image --steps 3 --kstats > gpurun_out/step_image.log 2>&1
DF_GEMM_SK=0 timeout 300 python tools/profile_step.py --config image --steps 3 --kstats >> gpurun_out/step_image.log 2>&1
