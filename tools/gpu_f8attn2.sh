cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_mxf8.py -q -s -k "qf8 or f8_vs or step or pipeline" > gpurun_out/f8a2_test.log 2>&1; echo rc=$? >> gpurun_out/f8a2_test.log
