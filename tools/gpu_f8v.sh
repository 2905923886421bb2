cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_mxf8.py -q -s -k "qf8 or f8_vs or step or pipeline or quant or gemm" > gpurun_out/f8v_test.log 2>&1; echo rc=$? >> gpurun_out/f8v_test.log
for r in 1 2; do for v in 2 1; do
  DF_ATTN_F8=$v timeout 300 python tools/profile_step.py --config image --precision fp8 --steps 8 2>&1 | sed "s/^/image f8lvl=$v run=$r /" >> gpurun_out/f8v_step.log
done; done
for s in image video; do timeout 300 python tools/attn_bench.py --shape $s --f8 2 --reps 10 --iters 3 >> gpurun_out/f8v_step.log 2>&1; done
