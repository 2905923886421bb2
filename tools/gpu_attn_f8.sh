# Standalone attention: bf16 vs e4m3 QK (R32) vs e4m3 QK + PV (R33), image / video self-attention
# shapes (f8 = 2 includes the V transpose-quantise launches), and ncu of the full-FP8 kernel at
# the video shape.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/attn_f8
for s in image video; do for f in 0 1 2; do
  timeout 300 python tools/attn_bench.py --shape $s --f8 $f --reps 10 --iters 3 >> gpurun_out/attn_f8/bench.log 2>&1
done; done
timeout 900 ncu --set full --clock-control none -k regex:attn_pp -s 1 -c 1 -o gpurun_out/attn_f8/f8 \
  python tools/attn_bench.py --shape video --f8 2 --iters 1 --reps 1 > gpurun_out/attn_f8/ncu.log 2>&1
ncu -i gpurun_out/attn_f8/f8.ncu-rep --page raw --csv > gpurun_out/attn_f8/raw.csv 2>&1
rm -f gpurun_out/attn_f8/f8.ncu-rep
