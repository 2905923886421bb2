cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --config video_i2v --dit-steps 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_video_i2v_4step.json 2> gpurun_out/bench_video_i2v.err
timeout 1500 python tools/handoff_stress.py --config image --dit-steps 8 --requests 24 --out gpurun_out/handoff_stress_image.json > gpurun_out/handoff_stress.log 2>&1
