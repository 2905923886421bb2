cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --t-per-gpu 2 --no-cpu-baseline > gpurun_out/bench_image_t2.json 2> gpurun_out/bench_image_t2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 750 -c 800 --csv --log-file gpurun_out/launches_image.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_pp -c 1 -o gpurun_out/ncu_pp_image python tools/attn_bench.py --shape image --iters 1 > gpurun_out/ncu_pp.log 2>&1
