#!/bin/bash
# compute-sanitizer passes over the tiny-shape kernel and pipeline tests (round 2 hygiene,
# VERDICT item 10): memcheck, racecheck (shared-memory hazards), synccheck (barrier misuse)
# and initcheck, each on the GEMM / attention / RMSNorm / handoff kernels at the tiny and mid
# shapes.  Run under gpurun from the repo root; logs land in gpurun_out/sanitize/.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="bruteforce or special_cases or rmsnorm or integer or stream_k or payload_hash"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 $CS --tool $tool --print-limit 20 --error-exitcode 9 \
    python -m pytest tests/test_gpu_kernels.py -q -x -k "$SEL" -p no:cacheprovider \
    > gpurun_out/sanitize/kernels_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize/kernels_$tool.log
done
for tool in memcheck synccheck; do
  timeout 1500 $CS --tool $tool --print-limit 20 --error-exitcode 9 \
    python -m pytest tests/test_gpu_dit.py -q -x -k "test_single_step_parity and cfg0" -p no:cacheprovider \
    > gpurun_out/sanitize/step_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize/step_$tool.log
  timeout 1500 $CS --tool $tool --print-limit 20 --error-exitcode 9 \
    python -m pytest tests/test_gpu_pipeline.py -q -x -k "test_pipeline_tiny_matches_oracle" -p no:cacheprovider \
    > gpurun_out/sanitize/pipeline_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize/pipeline_$tool.log
done
