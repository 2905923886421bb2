cd $GRAFT_REPO_ROOT
for s in video image; do
  for i in 4 5; do DF_ATTN_IMPL=$i DF_ATTN_POLY=9 timeout 120 python tools/attn_bench.py --shape $s | sed "s/^/nosoftmax /"; done
done > gpurun_out/attn_dbg9.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "stream_k or integer" > gpurun_out/pytest_sk.log 2>&1
