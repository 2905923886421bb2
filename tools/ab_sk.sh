# A/B of the stream-K schedule on the image step (bench kernel rates), run under gpurun.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/ab
for rep in 1 2; do
  timeout 600 python bench.py --video-requests 0 --no-cpu-baseline > gpurun_out/ab/base_$rep.json 2>/dev/null
  DF_GEMM_SK=1 timeout 600 python bench.py --video-requests 0 --no-cpu-baseline > gpurun_out/ab/sk_$rep.json 2>/dev/null
done
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k "stream_k or integer" > gpurun_out/ab/sk_tests.log 2>&1
