# Source-level ncu view of the image cross-attention launch (warp-state sampling per SASS line),
# exported on the box as CSV (the report itself stays there).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/ncu_src
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_pp -s 1 -c 1 \
  -o gpurun_out/ncu_src/attn_cross python tools/profile_step.py --config image --steps 1 --layers 1 > gpurun_out/ncu_src/log 2>&1
ncu -i gpurun_out/ncu_src/attn_cross.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_src/attn_cross_sass.csv 2>&1
ncu -i gpurun_out/ncu_src/attn_cross.ncu-rep --page details --csv > gpurun_out/ncu_src/attn_cross_details.csv 2>&1
ncu -i gpurun_out/ncu_src/attn_cross.ncu-rep --page raw --csv > gpurun_out/ncu_src/attn_cross_raw.csv 2>&1
rm -f gpurun_out/ncu_src/attn_cross.ncu-rep
ls -la gpurun_out/ncu_src
