cd $GRAFT_REPO_ROOT
for s in video image cross_image; do
  for i in 4 5; do DF_ATTN_IMPL=$i timeout 120 python tools/attn_bench.py --shape $s; DF_ATTN_IMPL=$i DF_ATTN_POLY=9 timeout 120 python tools/attn_bench.py --shape $s | sed "s/^/nosoftmax /"; done
done > gpurun_out/attn_conv.log 2>&1
for i in 4 5; do DF_ATTN_IMPL=$i DF_ATTN_POLY=2 timeout 120 python tools/attn_bench.py --shape video | sed "s/^/poly2 /"; done >> gpurun_out/attn_conv.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" > gpurun_out/pytest_attn.log 2>&1
