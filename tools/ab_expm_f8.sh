cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for r in 1 2; do for m in 2 1 5; do
  DF_ATTN_EXPM_F8=$m timeout 300 python tools/attn_bench.py --shape video --f8 2 --reps 5 --iters 3 2>&1 | sed "s/^/expm_f8=$m /" >> gpurun_out/ab_expm_f8.log
done; done
