cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/rep
for r in 1 2; do timeout 900 python bench.py --video-requests 0 --fp8-requests 0 --mxfp8-requests 0 > gpurun_out/rep/bench_image_$r.json 2> gpurun_out/rep/err_$r.txt; done
