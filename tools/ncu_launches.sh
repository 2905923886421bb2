# The launch list of the bench command (ncu --metrics gpu__time_duration.sum --clock-control none,
# B200_PROFILING.md): 800 launches of the image step after weight init, serialised and cold-cache
# (the SHARE per kernel class is comparable with bench.py, not the absolute times); summarised on
# the box.  Run under gpurun from the repo root.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 800 --csv \
  --log-file gpurun_out/launches_image_r02.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  --video-requests 0 --fp8-requests 0 --mxfp8-requests 0 > gpurun_out/launches_bench.log 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_image_r02.csv > gpurun_out/launches_image_r02_summary.json 2>&1
