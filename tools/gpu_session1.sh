# ad-hoc GPU session: pipeline tests, bench, step decomposition, GEMM microbench
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_scheduler.py -x -q > gpurun_out/pytest_pipe.log 2>&1; echo rc=$? >> gpurun_out/pytest_pipe.log
timeout 600 python bench.py > gpurun_out/bench_image.json 2> gpurun_out/bench_image.err
timeout 300 python tools/profile_step.py --config image --steps 4 > gpurun_out/step_image.log 2>&1
timeout 300 python tools/profile_step.py --config image --steps 4 --kstats >> gpurun_out/step_image.log 2>&1
timeout 300 python tools/gemm_bench.py > gpurun_out/gemm_bench.log 2>&1
DF_GEMM_NOEPI=1 timeout 300 python tools/gemm_bench.py --no-cublas | sed 's/^/noepi /' >> gpurun_out/gemm_bench.log 2>&1
