cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/pytest_kernels.log 2>&1; echo rc=$? >> gpurun_out/pytest_kernels.log
for tc in 1 2; do timeout 120 python tools/gemm_bench.py --no-cublas --tc $tc --only image_o; timeout 120 python tools/gemm_bench.py --no-cublas --tc $tc --only image_down; done > gpurun_out/gemm_sk.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_tc2 -c 2 -o gpurun_out/ncu_gemm_sk python tools/gemm_bench.py --no-cublas --tc 2 --only image_o > gpurun_out/ncu_gemm_sk.log 2>&1
