#!/bin/bash
# One B200 validation pass (run under gpurun from the repo root): the GPU parity suite, the
# driver's smoke(), the default bench line (image), the video line and the reference arm.
# Outputs land in gpurun_out/ (scratch); copy what should be judged into profiles/.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_image.json 2> gpurun_out/bench_image.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 1200 python bench.py --config video --steps 2 --warmup 3 > gpurun_out/bench_video.json 2> gpurun_out/bench_video.err
