cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_mxf8.py -q -x -s -k "qf8 or f8_vs or step or pipeline" > gpurun_out/f8a_test.log 2>&1; echo rc=$? >> gpurun_out/f8a_test.log
for v in 2 1; do
  DF_ATTN_F8=$v timeout 300 python tools/profile_step.py --config image --precision fp8 --steps 6 --kstats 2>&1 | grep "step_ms\|attn_self" | sed "s/^/image f8lvl=$v /" >> gpurun_out/f8a_step.log
  DF_ATTN_F8=$v timeout 600 python tools/profile_step.py --config video --layers 4 --precision fp8 --steps 3 --kstats 2>&1 | grep "step_ms\|attn_self" | sed "s/^/video f8lvl=$v /" >> gpurun_out/f8a_step.log
done
