# RMSNorm A/B (run under gpurun): standalone GB/s per implementation, the closed-form test
# through the default path, and the image bench line with the streaming vs warp-per-row kernel.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/ab
for impl in 0 1 2; do DF_RMS_IMPL=$impl timeout 300 python tools/rms_bench.py > gpurun_out/ab/rms_$impl.log 2>&1; done
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k "rmsnorm" > gpurun_out/ab/rms_test.log 2>&1
for rep in 1 2; do
  timeout 600 python bench.py --video-requests 0 --no-cpu-baseline > gpurun_out/ab/rms0_$rep.json 2>/dev/null
  DF_RMS_IMPL=1 timeout 600 python bench.py --video-requests 0 --no-cpu-baseline > gpurun_out/ab/rms1_$rep.json 2>/dev/null
done
