cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_pipeline.py -x -q -k "jitter or tiny" > gpurun_out/pytest_jit.log 2>&1
timeout 1500 python tools/handoff_stress.py --config image --dit-steps 8 --requests 24 --out gpurun_out/handoff_stress_image.json > gpurun_out/handoff_stress.log 2>&1
