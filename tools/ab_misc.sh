# A/B runs (under gpurun): programmatic dependent launch on every kernel (DF_PDL=1) and two
# co-located DiT instances per GPU (E:T:D 1:2:1), image workload, bf16 and FP8 lines.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/ab2
for rep in 1 2; do
  timeout 600 python bench.py --video-requests 0 --no-cpu-baseline > gpurun_out/ab2/base_$rep.json 2>/dev/null
  DF_PDL=1 timeout 600 python bench.py --video-requests 0 --no-cpu-baseline > gpurun_out/ab2/pdl_$rep.json 2>/dev/null
done
timeout 600 python bench.py --video-requests 0 --fp8-requests 0 --no-cpu-baseline --t-per-gpu 2 --steps 4 > gpurun_out/ab2/t2.json 2>/dev/null
