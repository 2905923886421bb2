cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" > gpurun_out/pytest_attn.log 2>&1
for s in video image cross_image cross_video; do timeout 120 python tools/attn_bench.py --shape $s; done > gpurun_out/attn_pp2.log 2>&1
