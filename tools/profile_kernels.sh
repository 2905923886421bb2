#!/bin/bash
# ncu evidence for profiles/ (run under gpurun, one GPU): the image step's launch list (the
# bench command, 800 launches after weight init) and --set full captures of the dominant
# kernels; summarise here with tools/ncu_summary.py.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 750 -c 800 --csv \
  --log-file gpurun_out/launches_image.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_pp -c 1 \
  -o gpurun_out/ncu_attn_video python tools/attn_bench.py --shape video --iters 1 > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tc2 -s 9 -c 1 \
  -o gpurun_out/ncu_mlp_up_image python tools/profile_step.py --config image --steps 1 --layers 2 > gpurun_out/ncu_mlp_up.log 2>&1
