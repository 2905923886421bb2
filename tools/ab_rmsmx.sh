# MXFP8 RMSNorm: streaming (default) vs one warp per row (DF_RMS_MX=1), parity then in-step A/B.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mxf8.py -q -x -k "step or pipeline" > gpurun_out/rmsmx_test.log 2>&1; echo rc=$? >> gpurun_out/rmsmx_test.log
for r in 1 2; do
  for v in "DF_RMS_MX=0" "DF_RMS_MX=1"; do
    env $v timeout 300 python tools/profile_step.py --config image --precision mxfp8 --steps 6 --kstats 2>&1 | grep "rmsnorm\|step_ms\|qkv\|mlp_up" | sed "s/^/$v run=$r /" >> gpurun_out/rmsmx_step.log
  done
done
env timeout 300 python tools/profile_step.py --config image --precision fp8 --steps 6 --kstats 2>&1 | sed "s/^/fp8 /" >> gpurun_out/rmsmx_step.log
