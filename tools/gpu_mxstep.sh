cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mxf8.py -q -x -s -k "step or pipeline" > gpurun_out/mxstep_test.log 2>&1; echo rc=$? >> gpurun_out/mxstep_test.log
# in-step A/B of the short-key cross-attention (attn_sk) vs attn_pp
for r in 1 2; do
  for sk in 1 0; do
    DF_ATTN_SK=$sk timeout 300 python tools/profile_step.py --config image --steps 8 --kstats 2>&1 | sed "s/^/sk=$sk run=$r /" >> gpurun_out/ab_sk_step.log
  done
done
timeout 900 python bench.py --fp8-requests 0 --video-requests 0 --steps 3 > gpurun_out/bench_mx.json 2> gpurun_out/bench_mx.err
