#!/bin/bash
# compute-sanitizer on the kernels added late in round 2: attn_sk (forced, small shapes), the
# MXFP8 quantiser / block-scaled GEMM and the e4m3-QK attention.  Logs in gpurun_out/sanitize2/.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/sanitize2
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  DF_ATTN_SK=2 timeout 1200 $CS --tool $tool --print-limit 20 --error-exitcode 9 \
    python -m pytest tests/test_gpu_attn_sk.py -q -x -k "vs_fp64 and 300" -p no:cacheprovider \
    > gpurun_out/sanitize2/attn_sk_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize2/attn_sk_$tool.log
  timeout 1200 $CS --tool $tool --print-limit 20 --error-exitcode 9 \
    python -m pytest tests/test_gpu_mxf8.py -q -x -k "quant_bit_exact and 256-128 or exact_on_small_integers and 256-256" -p no:cacheprovider \
    > gpurun_out/sanitize2/mxf8_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize2/mxf8_$tool.log
  timeout 1200 $CS --tool $tool --print-limit 20 --error-exitcode 9 \
    python -m pytest tests/test_gpu_fp8.py -q -x -k "qf8 and 2-300" -p no:cacheprovider \
    > gpurun_out/sanitize2/qf8_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize2/qf8_$tool.log
done
# ncu --set full of the MX GEMM (image QKV shape) and the e4m3-QK attention (video self-attention shape)
mkdir -p gpurun_out/ncu_r2b
timeout 600 ncu --set full --clock-control none -k regex:gemm_tc2 -s 1 -c 1 -o gpurun_out/ncu_r2b/mx_gemm \
  python tools/gemm_bench.py --mx --only image_qkv > gpurun_out/ncu_r2b/mx_gemm.log 2>&1
ncu -i gpurun_out/ncu_r2b/mx_gemm.ncu-rep --page raw --csv > gpurun_out/ncu_r2b/mx_gemm_raw.csv 2>&1
rm -f gpurun_out/ncu_r2b/mx_gemm.ncu-rep
