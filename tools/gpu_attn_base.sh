cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/g1.log
for s in cross_image cross_video image video; do timeout 300 python tools/attn_bench.py --shape $s --reps 20 --iters 5 --lib >> gpurun_out/g1.log 2>&1; done
timeout 300 python tools/attn_bench.py --shape cross_image --reps 1 --iters 5 >> gpurun_out/g1.log 2>&1
