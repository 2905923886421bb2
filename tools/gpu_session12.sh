cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_image.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_pair3 -c 1 -o gpurun_out/ncu_pair3_video python tools/attn_bench.py --shape video --iters 1 > gpurun_out/ncu_pair3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tc2_kernel -s 60 -c 6 -o gpurun_out/ncu_gemms_image python tools/profile_step.py --config image --steps 1 --layers 2 > gpurun_out/ncu_gemms.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:rmsnorm -s 5 -c 1 -o gpurun_out/ncu_rms_image python tools/profile_step.py --config image --steps 1 --layers 2 > gpurun_out/ncu_rms.log 2>&1
