# Source-level ncu of the short-key attention (attn_sk) on the image cross-attention shape,
# standalone (tools/attn_bench.py); plus the head-count sweep (fixed vs per-tile cost).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/ncu_sk
#for h in 12 24 48 96; do timeout 120 python tools/attn_bench.py --shape cross_image --H $h --reps 20 --iters 5 >> gpurun_out/ncu_sk/sweep.log 2>&1; done
#for h in 12 24 48 96; do DF_ATTN_SK=0 timeout 120 python tools/attn_bench.py --shape cross_image --H $h --reps 20 --iters 5 >> gpurun_out/ncu_sk/sweep.log 2>&1; done
DF_ATTN_SK=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_sk -s 1 -c 1 \
  -o gpurun_out/ncu_sk/sk python tools/attn_bench.py --shape cross_image --iters 2 --reps 1 > gpurun_out/ncu_sk/log 2>&1
ncu -i gpurun_out/ncu_sk/sk.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sk/sass.csv 2>&1
ncu -i gpurun_out/ncu_sk/sk.ncu-rep --page details --csv > gpurun_out/ncu_sk/details.csv 2>&1
ncu -i gpurun_out/ncu_sk/sk.ncu-rep --page raw --csv > gpurun_out/ncu_sk/raw.csv 2>&1
rm -f gpurun_out/ncu_sk/sk.ncu-rep
