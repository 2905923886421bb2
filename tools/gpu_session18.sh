cd $GRAFT_REPO_ROOT
timeout 300 python tools/profile_step.py --config image --steps 6 > gpurun_out/pdl.log 2>&1
DF_PDL=1 timeout 300 python tools/profile_step.py --config image --steps 6 >> gpurun_out/pdl.log 2>&1
timeout 300 python tools/profile_step.py --config image --steps 6 >> gpurun_out/pdl.log 2>&1
DF_PDL=1 timeout 300 python tools/profile_step.py --config image --steps 6 >> gpurun_out/pdl.log 2>&1
DF_PDL=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_pdl.json 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_nopdl.json 2>&1
