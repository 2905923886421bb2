cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_mxf8.py -q -x -s -k "qf8 or step or pipeline" > gpurun_out/qf8_test.log 2>&1; echo rc=$? >> gpurun_out/qf8_test.log
for p in fp8 mxfp8; do timeout 300 python tools/profile_step.py --config image --precision $p --steps 6 --kstats 2>&1 | sed "s/^/$p /" >> gpurun_out/qf8_step.log; done
for p in fp8 mxfp8; do timeout 600 python tools/profile_step.py --config video --layers 4 --precision $p --steps 3 --kstats 2>&1 | sed "s/^/video $p /" >> gpurun_out/qf8_step.log; done
for v in 0 1; do DF_RMS_MX=$v timeout 600 python tools/profile_step.py --config video --layers 4 --precision mxfp8 --steps 3 --kstats 2>&1 | grep "rmsnorm\|step_ms" | sed "s/^/video rmsmx=$v /" >> gpurun_out/qf8_step.log; done
