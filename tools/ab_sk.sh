# attn_sk S-ring depth A/B (DF_ATTN_SK_SD=2|3) against attn_pp (DF_ATTN_SK=0): parity tests with the
# default, then standalone and in-step timings (image full depth, video 4 layers).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attn_sk.py -q -x > gpurun_out/sk3_test.log 2>&1; echo rc=$? >> gpurun_out/sk3_test.log
DF_ATTN_SK_SD=2 timeout 600 python -m pytest tests/test_gpu_attn_sk.py -q -x >> gpurun_out/sk3_test.log 2>&1; echo rc=$? >> gpurun_out/sk3_test.log
for v in "DF_ATTN_SK_SD=3" "DF_ATTN_SK_SD=2" "DF_ATTN_SK=0"; do
  for s in cross_image cross_video; do env $v timeout 120 python tools/attn_bench.py --shape $s --reps 20 --iters 5 2>&1 | sed "s/^/$v /" >> gpurun_out/sk3_bench.log; done
done
for r in 1 2; do
  for v in "DF_ATTN_SK_SD=3" "DF_ATTN_SK_SD=2" "DF_ATTN_SK=0"; do
    env $v timeout 300 python tools/profile_step.py --config image --steps 6 --kstats 2>&1 | grep "attn_cross\|step_ms" | sed "s/^/$v run=$r /" >> gpurun_out/sk3_step.log
    env $v timeout 300 python tools/profile_step.py --config video --layers 4 --steps 3 --kstats 2>&1 | grep "attn_cross\|step_ms" | sed "s/^/video $v run=$r /" >> gpurun_out/sk3_step.log
  done
done
