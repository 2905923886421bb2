#!/bin/bash
# Final validation of the round: the parity suite (incl. production depth), smoke(), the default
# bench line (image + video / FP8 / MXFP8 sub-records), the reference arm, the FP8 / MXFP8 modes at
# the video shape, and the ncu launch list of the default bench command.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/final
bash tools/gpu_validate.sh
cp gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench_image.json gpurun_out/bench_ref.json gpurun_out/final/ 2>/dev/null
cp -r gpurun_out/depth gpurun_out/final/ 2>/dev/null
timeout 900 python bench.py --config video --precision fp8 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/final/bench_video_fp8.json 2> gpurun_out/final/bench_video_fp8.err
timeout 900 python bench.py --config video --precision mxfp8 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/final/bench_video_mxfp8.json 2> gpurun_out/final/bench_video_mxfp8.err
