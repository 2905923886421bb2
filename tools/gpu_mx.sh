cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python tools/mx_diag.py > gpurun_out/mx_diag.log 2>&1
timeout 900 python -m pytest tests/test_gpu_mxf8.py tests/test_gpu_fp8.py -q -x -s > gpurun_out/mx_test.log 2>&1; echo rc=$? >> gpurun_out/mx_test.log
timeout 600 python tools/gemm_bench.py --mx > gpurun_out/mx_bench.log 2>&1
