# ncu --set full captures of the image step's kernel classes (run under gpurun, one GPU): one
# request prologue + one denoising step with ONE layer (tools/profile_step.py), so the launch
# order is: prologue GEMMs (gemm_tc2 #0 txt1, #1 txt2, #2 cross K/V), then the step: #3 patch
# embed, #4 QKV, #5 O-proj, #6 cross-Q, #7 cross-O, #8 MLP up, #9 MLP down; attn_pp #0 self,
# #1 cross; RMSNorm #0 norm1, #1 cross pre-norm, #2 norm2.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/ncu
NCU="timeout 600 ncu --set full --import-source on --clock-control none -c 1"
P="python tools/profile_step.py --config image --steps 1 --layers 1"
$NCU -k regex:gemm_tc2 -s 5 -o gpurun_out/ncu/o_proj $P > gpurun_out/ncu/o_proj.log 2>&1
$NCU -k regex:gemm_tc2 -s 6 -o gpurun_out/ncu/cross_q $P > gpurun_out/ncu/cross_q.log 2>&1
$NCU -k regex:gemm_tc2 -s 7 -o gpurun_out/ncu/cross_o $P > gpurun_out/ncu/cross_o.log 2>&1
$NCU -k regex:gemm_tc2 -s 9 -o gpurun_out/ncu/mlp_down $P > gpurun_out/ncu/mlp_down.log 2>&1
$NCU -k regex:rmsnorm -s 0 -o gpurun_out/ncu/rmsnorm $P > gpurun_out/ncu/rmsnorm.log 2>&1
$NCU -k regex:attn_pp -s 1 -o gpurun_out/ncu/attn_cross $P > gpurun_out/ncu/attn_cross.log 2>&1
# summaries here (the reports are tens of MB each; gpurun copies back <= 64 MiB)
for k in o_proj cross_q cross_o mlp_down rmsnorm attn_cross; do
  [ -f gpurun_out/ncu/$k.ncu-rep ] && python tools/ncu_summary.py full gpurun_out/ncu/$k.ncu-rep > gpurun_out/ncu/$k.json 2>&1
  ncu -i gpurun_out/ncu/$k.ncu-rep --page details --csv > gpurun_out/ncu/${k}_details.csv 2>/dev/null
done
rm -f gpurun_out/ncu/*.ncu-rep
