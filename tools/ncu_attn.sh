cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_tc3 -c 1 -o gpurun_out/ncu_attn3_video python tools/attn_bench.py --shape video --iters 1 > gpurun_out/ncu_attn3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_tc3 -c 1 -o gpurun_out/ncu_attn3_cross python tools/attn_bench.py --shape cross_image --iters 1 >> gpurun_out/ncu_attn3.log 2>&1
