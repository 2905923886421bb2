cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
nproc > gpurun_out/host.txt; free -g >> gpurun_out/host.txt
DF_TEST_OUT=gpurun_out/depth timeout 2400 python -m pytest tests/test_gpu_depth.py tests/test_gpu_dit.py tests/test_gpu_pipeline.py -x -q -m gpu --durations=10 > gpurun_out/pytest_depth.log 2>&1; echo rc=$? >> gpurun_out/pytest_depth.log
