#!/bin/bash
# One B200 validation pass (run under gpurun from the repo root): the GPU parity suite, the
# driver's smoke(), the default bench line (image, with the video sub-record) and the reference
# arm.  DF_SKIP_DEPTH=1 leaves out the ~25 min production-depth parity tests (test_gpu_depth).
# Outputs land in gpurun_out/ (scratch); copy what should be judged into profiles/.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
IGN=""
[ "${DF_SKIP_DEPTH:-0}" = "1" ] && IGN="--ignore=tests/test_gpu_depth.py"
DF_TEST_OUT=gpurun_out/depth timeout 3000 python -m pytest tests -m gpu -x -q --durations=15 $IGN > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_image.json 2> gpurun_out/bench_image.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
