# attention -> projection dataflow: parity (step / layer / pipeline tests) then in-step A/B.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dit.py tests/test_gpu_pipeline.py -q -x > gpurun_out/df_test.log 2>&1; echo rc=$? >> gpurun_out/df_test.log
for r in 1 2; do
  for v in 1 0; do
    DF_DATAFLOW=$v timeout 300 python tools/profile_step.py --config image --steps 8 2>&1 | sed "s/^/df=$v run=$r /" >> gpurun_out/df_step.log
    DF_DATAFLOW=$v timeout 300 python tools/profile_step.py --config image --steps 4 --kstats 2>&1 | grep "o_proj\|cross_o\|attn" | sed "s/^/df=$v run=$r /" >> gpurun_out/df_step.log
  done
done
