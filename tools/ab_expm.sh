# A/B of the softmax exponential split (DF_ATTN_EXPM) on the attention shapes (standalone,
# 20 back-to-back launches per sample).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for m in 2 1 5 0 4 3; do
  for s in cross_image image video; do
    DF_ATTN_EXPM=$m timeout 200 python tools/attn_bench.py --shape $s --reps 10 --iters 3 2>&1 | sed "s/^/expm=$m /" >> gpurun_out/ab_expm.log
  done
done
