cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_tc3 -c 1 -o gpurun_out/ncu_attn3b_video python tools/attn_bench.py --shape video --iters 1 > gpurun_out/ncu_attn3b.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_image.json 2> gpurun_out/bench_image.err
timeout 300 python tools/profile_step.py --config image --steps 4 --kstats > gpurun_out/step_image.log 2>&1
