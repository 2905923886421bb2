cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_pipeline.py tests/test_gpu_scheduler.py -q --durations=10 > gpurun_out/pytest_mp.log 2>&1; echo rc=$? >> gpurun_out/pytest_mp.log
