cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dit.py -x -q > gpurun_out/pytest_k.log 2>&1; echo rc=$? >> gpurun_out/pytest_k.log
timeout 120 python tools/rms_bench.py > gpurun_out/rms.log 2>&1
timeout 300 python tools/gemm_bench.py --no-cublas > gpurun_out/gemm8.log 2>&1
timeout 300 python tools/profile_step.py --config image --steps 4 --kstats > gpurun_out/step_image.log 2>&1
