cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "variants" > gpurun_out/pytest_var.log 2>&1
for s in video image cross_image cross_video; do for i in 5 6; do DF_ATTN_IMPL=$i timeout 120 python tools/attn_bench.py --shape $s; done; done > gpurun_out/attn_pp.log 2>&1
